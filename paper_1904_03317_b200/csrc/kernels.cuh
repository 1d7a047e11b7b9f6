// sm_100a kernels of the local-smoothing GMG hot path (fp64, no tensor cores:
// the contractions are 3x3 / 5x5 per direction, not a GEMM).
//
//  fam_apply       y += K_l x over the cells of C_l, one block = FPB families of
//                  2^d sibling cells (the children of a refined level-(l-1) cell),
//                  thread per cell: register-resident sum-factorised Q_k Laplace
//                  (P:565-578), per-cell results combined per family patch in
//                  shared memory, patch-interior nodes stored exclusively, only
//                  family-boundary nodes scattered with fp64 atomics at L2
//  cell_apply      same operator over an explicit cell list (leaf cells of the
//                  leaf operator, level 0), thread per cell, atomic scatter
//  cell_diag       diagonal of the level operator
//  cell_load       b += f h^d (w (x) w (x) w) on leaf cells (f = const)
//  cheb_step       fused Chebyshev-Jacobi vector update + reset of the
//                  apply accumulator, double2 streaming
//  fam_restrict    d_{l-1} += P^T r, warp per family, r = d - K x computed on the
//                  fly for the V-cycle residual (edge rows included);
//                  each fine node is summed by the one family that owns it
//  fam_prolongate  x_l += P x_{l-1} on owned fine nodes (exclusive writes), or
//                  x_l[E] = (P x_{l-1})[E] (hanging / edge values, leaf operator)
//  dot / axpy      CG vector kernels with deterministic two-stage reductions
//
// Family patch table fam_dofs (AoS [n_fam][(2k+1)^d]): v >= 0: level DoF v owned
// (for transfers) by this family; v == -1: Dirichlet node; v <= -2: DoF -2-v
// owned by an earlier family.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <type_traits>

namespace gmg {
namespace dev {

// ------------------------------------------------------------- 1-D matrices
// Closed forms on the reference interval [0,1] with nodes {0, 1/k, .., 1}:
//   Q1: K = [[1,-1],[-1,1]],  M = [[1/3,1/6],[1/6,1/3]],  int phi = (1/2, 1/2)
//   Q2: K = 1/3 [[7,-8,1],[-8,16,-8],[1,-8,7]],  M = 1/30 [[4,2,-1],[2,16,2],[-1,2,4]],
//       int phi = (1/6, 2/3, 1/6)
// P(a, j): coarse basis j evaluated at fine patch coordinate a/(2k) of the parent.
template <int K> struct Q;
template <> struct Q<1> {
  static __host__ __device__ __forceinline__ constexpr double Km(int i, int j) { return i == j ? 1.0 : -1.0; }
  static __host__ __device__ __forceinline__ constexpr double Mm(int i, int j) { return i == j ? (1.0 / 3.0) : (1.0 / 6.0); }
  static __host__ __device__ __forceinline__ constexpr double w(int) { return 0.5; }
  static __host__ __device__ __forceinline__ constexpr double P(int a, int j) {
    return a == 1 ? 0.5 : ((a == 2 * j) ? 1.0 : 0.0);
  }
};
template <> struct Q<2> {
  static __host__ __device__ __forceinline__ constexpr double Km(int i, int j) {
    return (i == 1 && j == 1) ? 16.0 / 3.0 : ((i == 1 || j == 1) ? -8.0 / 3.0 : (i == j ? 7.0 / 3.0 : 1.0 / 3.0));
  }
  static __host__ __device__ __forceinline__ constexpr double Mm(int i, int j) {
    return (i == 1 && j == 1) ? 16.0 / 30.0 : ((i == 1 || j == 1) ? 2.0 / 30.0 : (i == j ? 4.0 / 30.0 : -1.0 / 30.0));
  }
  static __host__ __device__ __forceinline__ constexpr double w(int i) { return i == 1 ? (2.0 / 3.0) : (1.0 / 6.0); }
  // phi0 = 2t^2-3t+1, phi1 = 4t(1-t), phi2 = 2t^2-t at t = a/4
  static __host__ __device__ __forceinline__ constexpr double P(int a, int j) {
    return a == 0 ? (j == 0 ? 1.0 : 0.0)
         : a == 1 ? (j == 0 ? 0.375 : (j == 1 ? 0.75 : -0.125))
         : a == 2 ? (j == 1 ? 1.0 : 0.0)
         : a == 3 ? (j == 0 ? -0.125 : (j == 1 ? 0.75 : 0.375))
                  : (j == 2 ? 1.0 : 0.0);
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
template <int D, int K, typename T>
__device__ __forceinline__ void elem_apply(const T (&u)[Shape<D, K>::NN], T (&out)[Shape<D, K>::NN]) {
  constexpr int N = K + 1;
  if constexpr (D == 2) {
    T a[N * N], b[N * N];
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) {
        T sa = 0, sb = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          sa = fma((T)Q<K>::Km(x, q), u[y * N + q], sa);
          sb = fma((T)Q<K>::Mm(x, q), u[y * N + q], sb);
        }
        a[y * N + x] = sa;
        b[y * N + x] = sb;
      }
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) {
        T s = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          s = fma((T)Q<K>::Mm(y, q), a[q * N + x], s);
          s = fma((T)Q<K>::Km(y, q), b[q * N + x], s);
        }
        out[y * N + x] = s;
      }
  } else {
    constexpr int NN = N * N * N;
    T t1[NN], t2[NN];
    // z direction: t1 = M_z u, t2 = K_z u
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int yx = 0; yx < N * N; ++yx) {
        T s1 = 0, s2 = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          s1 = fma((T)Q<K>::Mm(z, q), u[q * N * N + yx], s1);
          s2 = fma((T)Q<K>::Km(z, q), u[q * N * N + yx], s2);
        }
        t1[z * N * N + yx] = s1;
        t2[z * N * N + yx] = s2;
      }
    // y direction: a = M_y t1, b = K_y t1 + M_y t2
    T a[NN], b[NN];
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int y = 0; y < N; ++y)
#pragma unroll
        for (int x = 0; x < N; ++x) {
          T sa = 0, sb = 0;
#pragma unroll
          for (int q = 0; q < N; ++q) {
            const int iq = z * N * N + q * N + x;
            sa = fma((T)Q<K>::Mm(y, q), t1[iq], sa);
            sb = fma((T)Q<K>::Km(y, q), t1[iq], sb);
            sb = fma((T)Q<K>::Mm(y, q), t2[iq], sb);
          }
          a[z * N * N + y * N + x] = sa;
          b[z * N * N + y * N + x] = sb;
        }
    // x direction: out = K_x a + M_x b
#pragma unroll
    for (int zy = 0; zy < N * N; ++zy)
#pragma unroll
      for (int x = 0; x < N; ++x) {
        T s = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          s = fma((T)Q<K>::Km(x, q), a[zy * N + q], s);
          s = fma((T)Q<K>::Mm(x, q), b[zy * N + q], s);
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

// patch coordinate of local node b of child c (compile-time after unrolling)
template <int D, int K>
__host__ __device__ __forceinline__ constexpr int patch_of(int c, int b) {
  constexpr int N = K + 1, NP1 = 2 * K + 1;
  int a = 0, mul = 1;
  for (int j = 0; j < D; ++j) {
    a += (((c >> j) & 1) * K + b % N) * mul;
    b /= N;
    mul *= NP1;
  }
  return a;
}

__device__ __forceinline__ int decode_dof(int v) { return v >= 0 ? v : (v <= -2 ? -2 - v : -1); }

// ------------------------------------------------------------- level operator
template <int D, int K> struct FamCfg { static constexpr int FPB = D == 3 ? 16 : 32; };

template <int D, int K, typename T>
__global__ void __launch_bounds__(FamCfg<D, K>::FPB * (1 << D))
fam_apply(int nfam, const int* __restrict__ fam_dofs, const double* __restrict__ coef, double scale,
          const T* __restrict__ x, T* __restrict__ y) {
  constexpr int NN = Shape<D, K>::NN, NP = Shape<D, K>::NP, NCH = Shape<D, K>::NCH;
  constexpr int NP1 = 2 * K + 1, N = K + 1;
  constexpr int FPB = FamCfg<D, K>::FPB, NT = FPB * NCH;
  __shared__ int sidx[FPB * NP];
  __shared__ T sout[NT * NN];
  const int tid = threadIdx.x;
  const long fam0 = (long)blockIdx.x * FPB;
  const int nf_here = (int)min((long)FPB, (long)nfam - fam0);
  // SoA patch table [NP][nfam]: row a holds the FPB families of this block contiguously
  for (int i = tid; i < FPB * NP; i += NT) {
    const int a = i / FPB, fl = i % FPB;
    sidx[fl * NP + a] = fl < nf_here ? __ldg(fam_dofs + (long)a * nfam + fam0 + fl) : -1;
  }
  __syncthreads();
  const int fl = tid / NCH, c = tid % NCH;
  if (fl < nf_here) {
    T u[NN], v[NN];
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      const int i = decode_dof(sidx[fl * NP + patch_of<D, K>(c, b)]);
      u[b] = i >= 0 ? __ldg(x + i) : T(0);
    }
    elem_apply<D, K, T>(u, v);
    const T s = (T)(coef ? scale * __ldg(coef + (fam0 + fl) * NCH + c) : scale);
#pragma unroll
    for (int b = 0; b < NN; ++b) sout[tid * NN + b] = s * v[b];
  }
  __syncthreads();
  for (int i = tid; i < nf_here * NP; i += NT) {
    const int fl2 = i / NP, a = i % NP;
    const int dof = decode_dof(sidx[i]);
    if (dof < 0) continue;
    int ad[3] = {a % NP1, (a / NP1) % NP1, D == 3 ? a / (NP1 * NP1) : 0};
    bool interior = true;
#pragma unroll
    for (int j = 0; j < D; ++j) interior &= (ad[j] > 0 && ad[j] < 2 * K);
    T sum = 0;
#pragma unroll
    for (int cc = 0; cc < NCH; ++cc) {
      bool in = true;
      int b = 0, mul = 1;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const int cj = (cc >> j) & 1;
        const int bj = ad[j] - cj * K;
        in &= (bj >= 0 && bj <= K);
        b += bj * mul;
        mul *= N;
      }
      if (in) sum += sout[(fl2 * NCH + cc) * NN + b];
    }
    if (interior) y[dof] = sum;          // only this family touches the node
    else atomicAdd(y + dof, sum);
  }
}

// Family-patch tensor form of the level operator.  On a family (2^d siblings of
// width h, one coefficient) the sum of the 2^d cell operators is itself a
// Kronecker sum over the (2k+1)^d patch: sum_i (x)_j (j == i ? Kt : Mt) with the
// 1-D matrices Kt, Mt assembled over the two children (P:575-577 applied to the
// patch).  Warp per family, one lane per 1-D line of the patch, 1-D passes
// through shared memory (7 passes in 3D, 4 in 2D); ~35% fewer DFMA than the 2^d
// separate cell operators and ~40 registers per thread instead of ~130.
template <int K>
__host__ __device__ __forceinline__ constexpr double Kt(int i, int j) {
  double s = 0.0;
  for (int e = 0; e < 2; ++e) {
    const int li = i - e * K, lj = j - e * K;
    if (li >= 0 && li <= K && lj >= 0 && lj <= K) s += Q<K>::Km(li, lj);
  }
  return s;
}
template <int K>
__host__ __device__ __forceinline__ constexpr double Mt(int i, int j) {
  double s = 0.0;
  for (int e = 0; e < 2; ++e) {
    const int li = i - e * K, lj = j - e * K;
    if (li >= 0 && li <= K && lj >= 0 && lj <= K) s += Q<K>::Mm(li, lj);
  }
  return s;
}

#ifndef TENSOR_WARPS_DEFAULT
#define TENSOR_WARPS_DEFAULT 4   // 2D kernels: warps per block (4: c2 V-cycle 0.634 -> 0.601 ms against 8; 2: 0.604)
#endif
constexpr int TENSOR_WARPS = TENSOR_WARPS_DEFAULT;

// one 1-D pass over `lines` lines of a 3-index array: in(i, q, o) -> out(i, p, o),
// out = sum_q M(p, q) in, with M = P (UP: q < N, p < NP1) or P^T (!UP)
template <int K, bool UP, int NI, int NO, typename T>
__device__ __forceinline__ void xfer_pass(int lane, const T* in, T* out, int si_in, int sq_in, int so_in,
                                          int si_out, int sp_out, int so_out) {
  constexpr int N = K + 1, NP1 = 2 * K + 1;
  constexpr int NQ = UP ? N : NP1, NPo = UP ? NP1 : N;
  for (int L = lane; L < NI * NO; L += 32) {
    const int i = L / NO, o = L % NO;
    T v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = in[i * si_in + q * sq_in + o * so_in];
#pragma unroll
    for (int p = 0; p < NPo; ++p) {
      T s = 0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        constexpr int dummy = 0;
        (void)dummy;
        const double m = UP ? Q<K>::P(p, q) : Q<K>::P(q, p);
        if (m != 0.0) s = fma((T)m, v[q], s);
      }
      out[i * si_out + p * sp_out + o * so_out] = s;
    }
  }
}

// fam_tensor_apply (3D) runs one block of TG_WARPS warps over FPB = 32 TG_WARPS
// / (2k+1)^2 families (5 for Q2, 14 for Q1), one thread per 1-D line of a
// patch: 125 of 128 lanes busy instead of 25 of 32 with a warp per family.
constexpr int TG_WARPS = 4;

// Transposition layouts (per family slot of the block): A holds the z-pass
// result for the y pass, B the y-pass result for the x pass (slot stride sab),
// N the x-pass result for the scatter along z lines (slot stride sn); index =
// cx x + cy y + cz z.  Chosen by exhaustive search so that every pass's
// shared-memory accesses (fp64 served per 16-lane half-warp over 16 bank pairs,
// fp32 in one pass over 32 banks; warps straddle two families) take the minimum
// number of wavefronts (tools/smem_layouts.py): A and B reach the ideal (2
// wavefronts per fp64 access of a warp, 1 per fp32 access); N cannot on every
// pass (the x-pass and z-pass line numberings swap the roles of y), it takes 25 %
// (fp64) / 38 % (fp32) more than the ideal on its two passes.
template <int K, typename T> struct PatchLayout {   // K = 1: natural order (27 nodes)
  static constexpr int ax = 1, ay = 2 * K + 1, az = (2 * K + 1) * (2 * K + 1);
  static constexpr int bx = 1, by = 2 * K + 1, bz = (2 * K + 1) * (2 * K + 1);
  static constexpr int nx = 1, ny = 2 * K + 1, nz = (2 * K + 1) * (2 * K + 1);
  static constexpr int sab = (2 * K + 1) * (2 * K + 1) * (2 * K + 1), sn = sab;
};
template <> struct PatchLayout<2, double> {   // wavefronts per 5 families: A 40+40, B 40+40, N 40+60
  static constexpr int ax = 1, ay = 5, az = 37, bx = 1, by = 33, bz = 5, sab = 185;
  static constexpr int nx = 1, ny = 5, nz = 25, sn = 125;
};
template <> struct PatchLayout<2, float> {    // A 20+20, B 20+20, N 35+20
  static constexpr int ax = 1, ay = 5, az = 37, bx = 1, by = 33, bz = 5, sab = 185;
  static constexpr int nx = 1, ny = 5, nz = 39, sn = 185;
};
template <int K> struct TensorCfg {
  static constexpr int NL = (2 * K + 1) * (2 * K + 1), FPB = 32 * TG_WARPS / NL;
};

// Epilogue modes of fam_tensor_apply: TA_APPLY y += K x (rows only this
// family touches -- R1 rows, rows < n_r1, and patch-interior nodes -- stored,
// the others reduced at L2); TA_CHEB_* in addition finish the Chebyshev-Jacobi
// step on the R1 rows (plan.hpp): dv = c1 dv + c2 D^-1 (g - K x),
// x += dv, with x_j taken from the gather; those rows never reach y.  Suffix:
// READ_DV / WRITE_DV.
// TA_CHEB_X1: the step after the first one from x = 0, where dv_0 = x_1 is not
// stored and is read from x (from the gather's registers in the epilogue).
// Where the fused epilogue requests g, D^-1, dv of its R1 rows: 0 with the x
// gather (80 registers), 1 after the z pass, 2 after the last pass (56).
#ifndef TA_LOAD_AT_DEFAULT
#define TA_LOAD_AT_DEFAULT 2
#endif
constexpr int TA_LOAD_AT = TA_LOAD_AT_DEFAULT;

// TA_CHEB_P01: the prolongation x += P x_{l-1} fused into the first step of the
// post-smoothing (TA_CHEB_01 on x + P x_{l-1}).  Every family computes P x_{l-1}
// on its whole patch from its parent's values: a fine node on a face, edge or
// corner shared with a family of another parent gets the same value bit for bit
// from either parent (the 1-D weights across the shared coordinate are exact
// picks, the others are the same weights on the same coarse values in the same
// order), so the gathered x + P x_{l-1} equals what warp_prolongate writes.  R1
// rows are finished here; for the other rows the transfer-owner family leaves
// P x_{l-1} in dv (dead before this step) and cheb_range<..., PRO> adds it.
enum : int { TA_APPLY = 0, TA_CHEB_01 = 1, TA_CHEB_11 = 2, TA_CHEB_10 = 3, TA_CHEB_00 = 4, TA_CHEB_X1 = 5,
             TA_CHEB_P01 = 6, TA_CHEB_Z1 = 7, TA_RES = 8 };
// TA_RES: the V-cycle's residual and restriction, d_{l-1} += P^T (d_l - K_l x_l)
// (P:427-437), in ONE pass over the level instead of the plain operator
// (t = K x, L2 reductions on shared rows), t's export-add and warp_restrict (which
// re-reads the patch rows, d and t).  By linearity P^T (d - K x) = sum over patches
// f of P_f^T (d|_{own f} - K_f x): each fine node's interpolation row is the same
// functional of the coarse DoFs from every parent whose closure holds it (continuity
// of the coarse Q_k space; the same exact-pick argument as TA_CHEB_P01), d enters
// once, through the node's transfer-owner patch (table entry >= 0, R26), and each
// patch's local operator result enters through its own parent(s).  So every patch
// restricts its own contribution -- P^T along z in registers on the scatter's z
// lines, then y and x through shared memory -- and adds (k+1)^3 (family) or
// (2k+1)^3 (grandfamily) coarse values at L2; y is the coarse defect d_{l-1}, g is
// d_l.  The level's t is neither written nor read.
// P over a grandfamily's two parents per direction: fine a in 0..4k, coarse j in 0..2k
template <int K>
__host__ __device__ __forceinline__ constexpr double P2(int a, int j) {
  const int c = a <= 2 * K ? 0 : 1, la = a - 2 * K * c, lj = j - K * c;
  return lj >= 0 && lj <= K ? Q<K>::P(la, lj) : 0.0;
}
// TA_CHEB_Z1: TA_CHEB_X1 without the preceding pass x_1 = c2_0 D^-1 g (the first step
// from x = 0): the gather forms x_1 = c0 D^-1 g itself on the owned rows (ghost rows:
// imported x_1, materialised on the owners' send rows), cheb_range<..., Z1> likewise

// the body of fam_tensor_apply for virtual block vb, shared memory passed in
// (s0, s1: TensorCfg<K>::NS entries each; cbf: FPB * ((k+1)^3 + 1) for TA_CHEB_P01), so
// that the persistent small-level kernel (small_vcycle) can run it too
template <int K, typename T> struct TensorSmem {
  static constexpr int NS = TensorCfg<K>::FPB * (PatchLayout<K, T>::sab > PatchLayout<K, T>::sn
                                                     ? PatchLayout<K, T>::sab : PatchLayout<K, T>::sn);
  // TA_CHEB_P01 per slot: the parent's (k+1)^3 values (+1 pad), then the separable
  // P passes' results: x pass (2k+1)(k+1)^2, y pass (2k+1)^2 (k+1)
  static constexpr int NCB1 = (K + 1) * (K + 1) * (K + 1) + 1 + (2 * K + 1) * (K + 1) * (K + 1) +
                              (2 * K + 1) * (2 * K + 1) * (K + 1);
  static constexpr int NCB = TensorCfg<K>::FPB * NCB1;
};
template <int K, typename T, int TM>
__device__ __forceinline__ void fam_tensor_body(long vb, T* __restrict__ s0, T* __restrict__ s1, T* __restrict__ cbf,
                 int nfam, const int* __restrict__ xfer, int row, const double* __restrict__ fcoef, double scale_,
                 const T* __restrict__ x, T* __restrict__ y, long n_r1, const T* __restrict__ g,
                 const T* __restrict__ Dinv, T* __restrict__ dv, T* xw,
                 double c1_, double c2_, const T* __restrict__ xc, int pf,
                 const int* __restrict__ flist, double c0_ = 0, long n_own = 0) {
  constexpr bool Z1 = TM == TA_CHEB_Z1;
  constexpr bool DVX = TM == TA_CHEB_X1 || Z1, PRO = TM == TA_CHEB_P01;
  constexpr bool RDV = TM == TA_CHEB_11 || TM == TA_CHEB_10 || DVX;
  constexpr bool WDV = TM == TA_CHEB_01 || TM == TA_CHEB_11 || DVX || PRO;
  constexpr bool RES = TM == TA_RES, CHEB = TM != TA_APPLY && !RES;
  constexpr int NP1 = 2 * K + 1, S2 = NP1 * NP1, NL = TensorCfg<K>::NL, FPB = TensorCfg<K>::FPB;
  using LY = PatchLayout<K, T>;
  constexpr int NS = FPB * (LY::sab > LY::sn ? LY::sab : LY::sn);
  (void)NS;
  constexpr int NCB1 = TensorSmem<K, T>::NCB1;   // PRO: the parents' values and the P passes, per slot
  const int slot = threadIdx.x / NL, lane = threadIdx.x % NL;   // lane: line of the family's patch
  const long fi = vb * FPB + slot;
  const bool act = slot < FPB && fi < nfam;
  // flist: the families not covered by grandfamily patches (gfam_tensor_apply)
  const long f = flist ? (act ? (long)__ldg(flist + fi) : 0) : fi;
  if (pf > 0 && !flist) {   // the patch rows of the block one resident wave ahead -> L2 (their first touch is DRAM latency)
    const long fb = (vb + pf) * FPB;
    const long bytes = (long)FPB * row * 4, off = (long)threadIdx.x * 128;
    if (fb < nfam && off < bytes && fb * row * 4 + off < (long)nfam * row * 4)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(xfer + fb * (long)row) + off));
  }
  const int* rp = xfer + (act ? f : 0) * (long)row;
  T* const a0 = s0 + (act ? slot : 0) * LY::sab;
  T* const a1 = s1 + (act ? slot : 0) * LY::sab;
  T* const n0 = s0 + (act ? slot : 0) * LY::sn;
  const T scale = (T)(act && fcoef ? scale_ * __ldg(fcoef + f) : scale_);   // config 4: one coefficient per family (levels >= 3)
  int gi[NP1];           // the z-line DoFs of this lane, reused by the scatter
  T ukeep[NP1];          // the gathered x values (x_j of the fused Chebyshev rows)
  T pg[NP1], pd[NP1], pv[NP1];   // fused modes: g, D^-1, dv of the R1 rows
  T inc[PRO ? NP1 : 1];          // PRO: (P x_{l-1}) on the z line
  int own = 0;                   // PRO: bit z = the family is the row's transfer owner
  T u[NP1];
  // PRO: the parent's coarse indices requested first (the coarse gather then goes
  // out with the fine one)
  constexpr int NCL = PRO ? ((K + 1) * (K + 1) * (K + 1) + NL - 1) / NL : 1;
  int cidx[NCL];
  if (PRO && act) {
#pragma unroll
    for (int j = 0; j < NCL; ++j)
      cidx[j] = lane + j * NL < (K + 1) * (K + 1) * (K + 1) ? __ldg(rp + NP1 * S2 + lane + j * NL) : -1;
  }
  if (act) {             // z lines: lane = (px, py), gathered straight into registers
#pragma unroll
    for (int z = 0; z < NP1; ++z) {
      const int e = __ldg(rp + z * S2 + lane);
      gi[z] = decode_dof(e);
      if ((PRO || RES) && e >= 0) own |= 1 << z;
    }
#pragma unroll
    for (int z = 0; z < NP1; ++z) {
      const int i = gi[z];
      if (Z1) u[z] = i < 0 ? T(0) : (i < n_own ? (T)c0_ * __ldg(Dinv + i) * __ldg(g + i) : __ldg(x + i));
      else u[z] = i >= 0 ? __ldg(x + i) : T(0);
    }
  }
  if constexpr (PRO) {
    // P x_{l-1} on this thread's z line: the parent's values are staged once per
    // family, then (P (x) P (x) P) by separable passes in warp_prolongate's order
    // (x, then y, then z; fma chains over ascending coarse index; a zero weight
    // adds an exact 0), so the result is its bit pattern
    constexpr int N = K + 1, NC = N * N * N, NPT = NP1 * NP1 * NP1;
    if (act) {             // 27 values, 25 lines
#pragma unroll
      for (int j = 0; j < NCL; ++j)
        if (lane + j * NL < NC) cbf[slot * NCB1 + lane + j * NL] = cidx[j] >= 0 ? __ldg(xc + cidx[j]) : T(0);
    }
    __syncthreads();
    // separable: x pass over the parent's (y, z) lines, y pass over (x, z), z pass
    // on this thread's z line -- each an fma chain over ascending coarse index, as
    // warp_prolongate (x, then y, then z), so the bits are the same
    T* const cbs = cbf + (act ? slot : 0) * NCB1;
    T* const bxs = cbs + NC + 1;                  // [c][b][px]
    T* const bys = bxs + NP1 * N * N;             // [c][py][px]
    if (act && lane < N * N) {
      const int b = lane % N, c = lane / N;
      T v[N];
#pragma unroll
      for (int a = 0; a < N; ++a) v[a] = cbs[a + N * b + N * N * c];
#pragma unroll
      for (int p = 0; p < NP1; ++p) {
        T sx = T(0);
#pragma unroll
        for (int a = 0; a < N; ++a) sx = fma((T)Q<K>::P(p, a), v[a], sx);
        bxs[p + NP1 * b + NP1 * N * c] = sx;
      }
    }
    __syncthreads();
    if (act && lane < NP1 * N) {
      const int qx = lane % NP1, c = lane / NP1;
      T v[N];
#pragma unroll
      for (int b = 0; b < N; ++b) v[b] = bxs[qx + NP1 * b + NP1 * N * c];
#pragma unroll
      for (int p = 0; p < NP1; ++p) {
        T sy = T(0);
#pragma unroll
        for (int b = 0; b < N; ++b) sy = fma((T)Q<K>::P(p, b), v[b], sy);
        bys[qx + NP1 * p + S2 * c] = sy;
      }
    }
    __syncthreads();
    if (act) {
      T w[N];
#pragma unroll
      for (int c = 0; c < N; ++c) w[c] = bys[lane + S2 * c];
#pragma unroll
      for (int z = 0; z < NP1; ++z) {
        T sz = T(0);
#pragma unroll
        for (int c = 0; c < N; ++c)
          if (Q<K>::P(z, c) != 0.0) sz = fma((T)Q<K>::P(z, c), w[c], sz);
        inc[z] = sz;
      }
    }
  }
  if (act) {
    if constexpr (PRO) {   // the gather above is in flight while P x_{l-1} is formed
#pragma unroll
      for (int z = 0; z < NP1; ++z) {
        if (gi[z] >= 0) u[z] = u[z] + inc[z];    // = warp_prolongate's old + fine
        // P x_{l-1} of a streamed row this family transfer-owns -> dv now (cheb_range<PRO>)
        if (((own >> z) & 1) && gi[z] >= n_r1) dv[gi[z]] = inc[z];
      }
    }
#pragma unroll
    for (int z = 0; z < NP1; ++z) ukeep[z] = u[z];
    if (CHEB && TA_LOAD_AT == 0) {   // requested with the gather: one memory round trip
#pragma unroll
      for (int z = 0; z < NP1; ++z) {
        const int i = gi[z];
        pg[z] = pd[z] = pv[z] = T(0);
        if (i >= 0 && i < n_r1) {
          pg[z] = __ldg(g + i);
          pd[z] = __ldg(Dinv + i);
          if (RDV && !DVX) pv[z] = dv[i];
        }
      }
    }
#pragma unroll
    for (int z = 0; z < NP1; ++z) {
      T t1 = 0, t2 = 0;
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        if (Mt<K>(z, q) != 0.0) t1 = fma((T)Mt<K>(z, q), u[q], t1);
        if (Kt<K>(z, q) != 0.0) t2 = fma((T)Kt<K>(z, q), u[q], t2);
      }
      const int ia = LY::ax * (lane % NP1) + LY::ay * (lane / NP1) + LY::az * z;   // layout A
      a0[ia] = t1;
      a1[ia] = t2;
    }
    if (CHEB && TA_LOAD_AT == 1) {   // in flight across the y and x passes
#pragma unroll
      for (int z = 0; z < NP1; ++z) {
        const int i = gi[z];
        pg[z] = pd[z] = pv[z] = T(0);
        if (i >= 0 && i < n_r1) {
          pg[z] = __ldg(g + i);
          pd[z] = __ldg(Dinv + i);
          if (RDV && !DVX) pv[z] = dv[i];
        }
      }
    }
  }
  __syncthreads();
  T t1[NP1], t2[NP1];
  const int px = lane % NP1, pz = lane / NP1;   // y lines: lane = (px, pz)
  if (act) {
    const int ba = LY::ax * px + LY::az * pz;
#pragma unroll
    for (int q = 0; q < NP1; ++q) {
      t1[q] = a0[ba + LY::ay * q];
      t2[q] = a1[ba + LY::ay * q];
    }
  }
  __syncthreads();       // layout B overwrites layout A
  if (act) {
    const int bb_ = LY::bx * px + LY::bz * pz;
#pragma unroll
    for (int yy = 0; yy < NP1; ++yy) {
      T a = 0, bb = 0;
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        if (Mt<K>(yy, q) != 0.0) {
          a = fma((T)Mt<K>(yy, q), t1[q], a);
          bb = fma((T)Mt<K>(yy, q), t2[q], bb);
        }
        if (Kt<K>(yy, q) != 0.0) bb = fma((T)Kt<K>(yy, q), t1[q], bb);
      }
      a0[bb_ + LY::by * yy] = a;   // layout B
      a1[bb_ + LY::by * yy] = bb;
    }
  }
  __syncthreads();
  T out[NP1];
  if (act) {             // x lines: lane = (py, pz)
    const int bx = LY::by * (lane % NP1) + LY::bz * (lane / NP1);
#pragma unroll
    for (int q = 0; q < NP1; ++q) {
      t1[q] = a0[bx + LY::bx * q];
      t2[q] = a1[bx + LY::bx * q];
    }
#pragma unroll
    for (int xx = 0; xx < NP1; ++xx) {
      T o = 0;
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        if (Kt<K>(xx, q) != 0.0) o = fma((T)Kt<K>(xx, q), t1[q], o);
        if (Mt<K>(xx, q) != 0.0) o = fma((T)Mt<K>(xx, q), t2[q], o);
      }
      out[xx] = scale * o;
    }
  }
  // x-line results -> layout N, then the scatter runs along the z lines of the
  // gather with the DoF indices still in registers
  __syncthreads();       // every lane has read layout B
  if (act) {
    const int bn = LY::ny * (lane % NP1) + LY::nz * (lane / NP1);
#pragma unroll
    for (int q = 0; q < NP1; ++q) n0[bn + LY::nx * q] = out[q];
  }
  if (CHEB && TA_LOAD_AT == 2 && act) {   // the epilogue's loads after the passes (fewer live registers)
#pragma unroll
    for (int z = 0; z < NP1; ++z) {
      const int i = gi[z];
      pg[z] = pd[z] = pv[z] = T(0);
      if (i >= 0 && i < n_r1) {
        pg[z] = __ldg(g + i);
        pd[z] = __ldg(Dinv + i);
        if (RDV && !DVX) pv[z] = dv[i];
      }
    }
  }
  if (RES && act) {   // d on the patch nodes this patch restricts (transfer owner, R26); issued here:
    // requesting it after the z pass was slower (c5 level 10: 1191-1208 vs 1030-1042 us)
#pragma unroll
    for (int z = 0; z < NP1; ++z) pg[z] = ((own >> z) & 1) ? __ldg(g + gi[z]) : T(0);
  }
  __syncthreads();
  if constexpr (RES) {
    // r = d|_own - K_f x on the z line (N read), P^T along z in registers -> s1 as
    // [jz][py][px]; y pass -> s0 as [jz][jy][px]; x pass -> (k+1)^3 coarse values
    constexpr int N = K + 1;
    T* const c1s = s1 + (act ? slot : 0) * LY::sab;
    if (act) {
      const int py = lane / NP1;
      const int bn = LY::nx * px + LY::ny * py;
      T rc[N];
#pragma unroll
      for (int c = 0; c < N; ++c) rc[c] = T(0);
#pragma unroll
      for (int z = 0; z < NP1; ++z) {
        if (gi[z] < 0) continue;
        const T r = pg[z] - n0[bn + LY::nz * z];
#pragma unroll
        for (int c = 0; c < N; ++c)
          if (Q<K>::P(z, c) != 0.0) rc[c] = fma((T)Q<K>::P(z, c), r, rc[c]);
      }
#pragma unroll
      for (int c = 0; c < N; ++c) c1s[lane + S2 * c] = rc[c];
    }
    __syncthreads();     // every lane has read layout N (s0)
    T* const c0s = s0 + (act ? slot : 0) * LY::sab;
    if (act && lane < NP1 * N) {   // y lines: (qx, jz)
      const int qx = lane % NP1, jz = lane / NP1;
      T w[NP1];
#pragma unroll
      for (int q = 0; q < NP1; ++q) w[q] = c1s[qx + NP1 * q + S2 * jz];
#pragma unroll
      for (int jy = 0; jy < N; ++jy) {
        T a = T(0);
#pragma unroll
        for (int q = 0; q < NP1; ++q)
          if (Q<K>::P(q, jy) != 0.0) a = fma((T)Q<K>::P(q, jy), w[q], a);
        c0s[qx + NP1 * jy + NP1 * N * jz] = a;
      }
    }
    __syncthreads();
    if (act && lane < N * N) {     // x lines: (jy, jz)
      const int jy = lane % N, jz = lane / N;
      T w[NP1];
#pragma unroll
      for (int q = 0; q < NP1; ++q) w[q] = c0s[q + NP1 * jy + NP1 * N * jz];
      constexpr int NPT = NP1 * NP1 * NP1;
#pragma unroll
      for (int jx = 0; jx < N; ++jx) {
        T a = T(0);
#pragma unroll
        for (int q = 0; q < NP1; ++q)
          if (Q<K>::P(q, jx) != 0.0) a = fma((T)Q<K>::P(q, jx), w[q], a);
        const int ci = __ldg(rp + NPT + jx + N * jy + N * N * jz);
        if (ci >= 0) atomicAdd(y + ci, a);
      }
    }
    return;
  }
  if (act) {
    const int py = lane / NP1;
    const bool inner = px > 0 && px < 2 * K && py > 0 && py < 2 * K;
    const int bn = LY::nx * px + LY::ny * py;
#pragma unroll
    for (int z = 0; z < NP1; ++z) {
      const int i = gi[z];
      if (i < 0) continue;
      const T v = n0[bn + LY::nz * z];
      if (CHEB && i < n_r1) {
        // complete row of an R1 node: Chebyshev step right here
        T dd = (T)c2_ * pd[z] * (pg[z] - v);
        if (RDV) dd = fma((T)c1_, DVX ? ukeep[z] : pv[z], dd);
        if (WDV) dv[i] = dd;
        xw[i] = ukeep[z] + dd;
      } else {
        if (i < n_r1 || (inner && z > 0 && z < 2 * K)) y[i] = v;   // only this family touches the node
        else atomicAdd(y + i, v);
      }
    }
  }
}

template <int K, typename T, int TM = TA_APPLY>
__global__ void __launch_bounds__(32 * TG_WARPS)
fam_tensor_apply(int nfam, const int* __restrict__ xfer, int row, const double* __restrict__ fcoef, double scale_,
                 const T* __restrict__ x, T* __restrict__ y, long n_r1 = 0, const T* __restrict__ g = nullptr,
                 const T* __restrict__ Dinv = nullptr, T* __restrict__ dv = nullptr, T* xw = nullptr,
                 double c1_ = 0, double c2_ = 0, const T* __restrict__ xc = nullptr, int pf = 0,
                 const int* __restrict__ flist = nullptr, double c0_ = 0, long n_own = 0) {
  using SM = TensorSmem<K, T>;
  __shared__ T s0[SM::NS], s1[SM::NS];
  __shared__ T cb[TM == TA_CHEB_P01 ? SM::NCB : 1];
  fam_tensor_body<K, T, TM>(blockIdx.x, s0, s1, cb, nfam, xfer, row, fcoef, scale_, x, y, n_r1, g, Dinv, dv, xw, c1_,
                            c2_, xc, pf, flist, c0_, n_own);
}

// fam_col_apply: the plain operator (TA_APPLY) on family patches with one thread
// per x-column of the patch (2k+1 threads per family, each holding the (2k+1)^2
// nodes (y, z) of its column in registers).  The same Kronecker sum as
// fam_tensor_apply, ordered so that two of the three 1-D passes run in registers:
//   c1 = (M_y (x) M_z) u,  c2 = (K_y (x) M_z + M_y (x) K_z) u   per column (registers),
//   out = K_x c1 + M_x c2                                        along x lines (shared),
// i.e. one transposition of two arrays and one back instead of fam_tensor_apply's
// three (2 + 2 + 1 arrays): 6 shared-memory accesses per patch node instead of 10.
// Gather and scatter run along the columns with the DoF indices in registers
// (lanes (family, px) read x-consecutive nodes, as fam_tensor_apply's z lines do).
// Shared layout, per array: node (x, j = y + (2k+1) z) of block family f at
// j S + (2k+1) f + x with S = (2k+1) FPC + 1 = 1 mod 16: the column writes and
// reads hit consecutive addresses (thread t = (2k+1) f + px), the x-line reads
// of thread (f, r) -- lines (y = r, z) -- hit r + 5 f + const (mod 16): no bank
// conflicts on any pass.  The x-line thread writes its result over the c1 entries
// it alone read.  FPC families per block.
template <int K, int FPC> struct ColCfg {
  static constexpr int NP1 = 2 * K + 1, NJ = NP1 * NP1, THREADS = NP1 * FPC, S = NP1 * FPC + 1;
  static constexpr int NS = NJ * S;
};
template <int K, typename T, int FPC>
__global__ void __launch_bounds__(ColCfg<K, FPC>::THREADS)
fam_col_apply(int nfam, const int* __restrict__ xfer, int row, const double* __restrict__ fcoef, double scale_,
              const T* __restrict__ x, T* __restrict__ y, long n_r1, int pf, const int* __restrict__ flist) {
  using C = ColCfg<K, FPC>;
  constexpr int NP1 = C::NP1, NJ = C::NJ, S = C::S;
  extern __shared__ __align__(16) unsigned char col_smem[];
  T* const c1s = reinterpret_cast<T*>(col_smem);
  T* const c2s = c1s + C::NS;
  const int t = threadIdx.x, fl = t / NP1, px = t % NP1;
  const long fi = (long)blockIdx.x * FPC + fl;
  const bool act = fi < nfam;
  const long f = flist ? (act ? (long)__ldg(flist + fi) : 0) : fi;
  if (pf > 0 && !flist) {   // the patch rows of the block one resident wave ahead -> L2
    const long fb = ((long)blockIdx.x + pf) * FPC;
    const long bytes = (long)FPC * row * 4, off = (long)t * 128;
    if (fb < nfam && off < bytes && fb * row * 4 + off < (long)nfam * row * 4)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(xfer + fb * (long)row) + off));
  }
  const int* rp = xfer + (act ? f : 0) * (long)row;
  int gi[NJ];
  T u[NJ];
  if (act) {
#pragma unroll
    for (int j = 0; j < NJ; ++j) gi[j] = decode_dof(__ldg(rp + j * NP1 + px));   // node (px, y, z), j = y + NP1 z
#pragma unroll
    for (int j = 0; j < NJ; ++j) u[j] = gi[j] >= 0 ? __ldg(x + gi[j]) : T(0);
    // z pass per y row: m = M_z u, k = K_z u
    T m[NJ], kz[NJ];
#pragma unroll
    for (int yy = 0; yy < NP1; ++yy)
#pragma unroll
      for (int z = 0; z < NP1; ++z) {
        T a = 0, b = 0;
#pragma unroll
        for (int q = 0; q < NP1; ++q) {
          if (Mt<K>(z, q) != 0.0) a = fma((T)Mt<K>(z, q), u[yy + NP1 * q], a);
          if (Kt<K>(z, q) != 0.0) b = fma((T)Kt<K>(z, q), u[yy + NP1 * q], b);
        }
        m[yy + NP1 * z] = a;
        kz[yy + NP1 * z] = b;
      }
    // y pass per z: c1 = M_y m, c2 = K_y m + M_y k -> shared
#pragma unroll
    for (int z = 0; z < NP1; ++z)
#pragma unroll
      for (int yy = 0; yy < NP1; ++yy) {
        T a = 0, b = 0;
#pragma unroll
        for (int q = 0; q < NP1; ++q) {
          if (Mt<K>(yy, q) != 0.0) {
            a = fma((T)Mt<K>(yy, q), m[q + NP1 * z], a);
            b = fma((T)Mt<K>(yy, q), kz[q + NP1 * z], b);
          }
          if (Kt<K>(yy, q) != 0.0) b = fma((T)Kt<K>(yy, q), m[q + NP1 * z], b);
        }
        const int j = yy + NP1 * z;
        c1s[j * S + t] = a;
        c2s[j * S + t] = b;
      }
  }
  __syncthreads();
  if (act) {   // x lines (y = px, z): out = scale (K_x c1 + M_x c2), over c1
    const T scale = (T)(fcoef ? scale_ * __ldg(fcoef + f) : scale_);
#pragma unroll
    for (int z = 0; z < NP1; ++z) {
      const int base = (px + NP1 * z) * S + NP1 * fl;
      T a[NP1], b[NP1];
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        a[q] = c1s[base + q];
        b[q] = c2s[base + q];
      }
#pragma unroll
      for (int xx = 0; xx < NP1; ++xx) {
        T o = 0;
#pragma unroll
        for (int q = 0; q < NP1; ++q) {
          if (Kt<K>(xx, q) != 0.0) o = fma((T)Kt<K>(xx, q), a[q], o);
          if (Mt<K>(xx, q) != 0.0) o = fma((T)Mt<K>(xx, q), b[q], o);
        }
        c1s[base + xx] = scale * o;
      }
    }
  }
  __syncthreads();
  if (act) {   // scatter along the column: rows only this family touches stored, the others reduced at L2
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int i = gi[j];
      if (i < 0) continue;
      const T v = c1s[j * S + t];
      const int yy = j % NP1, z = j / NP1;
      const bool inner = px > 0 && px < 2 * K && yy > 0 && yy < 2 * K && z > 0 && z < 2 * K;
      if (i < n_r1 || inner) y[i] = v;
      else atomicAdd(y + i, v);
    }
  }
}
template <int K, typename T, int FPC>
constexpr size_t col_smem_bytes() { return 2 * sizeof(T) * ColCfg<K, FPC>::NS; }

// ------------------------------------------------------------- grandfamily patches
// gfam_tensor_apply: the level operator on the (4k+1)^3 patch of a complete
// grandfamily -- the 64 level-l cells below one level-(l-2) cell G all of whose 8
// children are refined -- as ONE Kronecker sum with the 1-D matrices assembled
// over four cells (Kt4, Mt4).  Against eight separate family patches this
// gathers 729 instead of 1000 values (Q2), reads 729 instead of 1000 index
// entries, transposes 27 % fewer values through shared memory, and its 7^3
// patch-interior nodes (343 of the 512 rows the 64 cells own) are complete rows:
// stored / finished by the fused Chebyshev epilogue instead of reduced at L2 and
// streamed.  Thick refined regions (config 5's shell, config 4's corner) consist
// mostly of complete grandfamilies; thin ones (config 3's finest level) have none
// and keep the family kernel.  Epilogue modes as fam_tensor_apply (TA_*).
// Table gxfer [n_gf][GF_ROW]: 729 fine patch entries (x fastest; v >= 0: this
// grandfamily holds the node's transfer-owner family, v <= -2: DoF -2-v owned by
// another family, -1: Dirichlet), then the 125 level-(l-1) DoFs of G's family
// patch (the 8 parents' nodes; used by TA_CHEB_P01).
template <int K>
__host__ __device__ __forceinline__ constexpr double Kt4(int i, int j) {
  double s = 0.0;
  for (int e = 0; e < 4; ++e) {
    const int li = i - e * K, lj = j - e * K;
    if (li >= 0 && li <= K && lj >= 0 && lj <= K) s += Q<K>::Km(li, lj);
  }
  return s;
}
template <int K>
__host__ __device__ __forceinline__ constexpr double Mt4(int i, int j) {
  double s = 0.0;
  for (int e = 0; e < 4; ++e) {
    const int li = i - e * K, lj = j - e * K;
    if (li >= 0 && li <= K && lj >= 0 && lj <= K) s += Q<K>::Mm(li, lj);
  }
  return s;
}

// Grandfamilies per block (SLOTS) and threads: 1 -> 96 (81 lanes busy), 2 -> 192,
// 3 -> 256 (243 busy); the minimum-blocks bound caps registers at ~80.
#ifndef GF_LOAD_AT_DEFAULT
#define GF_LOAD_AT_DEFAULT 2
#endif
constexpr int GF_LOAD_AT = GF_LOAD_AT_DEFAULT;   // fused epilogue loads: 1 after the z pass, 2 after the x pass, 3 per row in the scatter
static_assert(GF_LOAD_AT >= 1 && GF_LOAD_AT <= 3, "gfam_tensor_apply has no epilogue-load placement 0");
#ifndef GF_REG_CAP
#define GF_REG_CAP 80
#endif
template <int SLOTS> struct GfBlock {
  static constexpr int THREADS = SLOTS == 1 ? 96 : (SLOTS == 2 ? 192 : 256);
  static constexpr int MIN_BLOCKS = 65536 / (THREADS * GF_REG_CAP);
};
template <int K> struct GfShape {
  static constexpr int N1 = 4 * K + 1, NL = N1 * N1, NP = N1 * N1 * N1;
  static constexpr int NCP = (2 * K + 1) * (2 * K + 1) * (2 * K + 1);   // G's family patch one level up
  static constexpr int ROW = NP + NCP;
  // TA_CHEB_P01 per slot: G's coarse patch (+1 pad), the x pass (4k+1)(2k+1)^2 and the
  // y pass (4k+1)^2 (2k+1) of the separable prolongation
  static constexpr int NCB = NCP + 1 + N1 * (2 * K + 1) * (2 * K + 1) + N1 * N1 * (2 * K + 1);
};
// Transposition layouts (index = cx x + cy y + cz z, per slot).  fp64 shared
// memory serves a half-warp per pass over 16 bank pairs, so an access whose 16
// lanes hit 16 distinct addresses mod 16 takes the minimum of one wavefront per
// half-warp.  Lanes number a line as L = a + 9 b (a, b its two coordinates); the
// strides (1, 9) and (9, 1) (mod 16) are both injective on 16 consecutive L, so
// for Q2 (9^3 patch):
//   A  z-pass store (px, py), y-pass load (px, pz):  ax = 1, ay = 9,  az = 89
//   B  y-pass store (px, pz), x-pass load (py, pz):  bx = 9, by = 89, bz = 1
//   N  x-pass store (py, pz), scatter load (px, py):  nx = 1, ny = 9,  nz = 81
// every pass is conflict-free (up to the half-warps straddling two slots; the
// slot stride is 1 mod 16).  N reuses the first buffer.  Other K: natural order.
template <int K> struct GfLayout {
  static constexpr int N1 = 4 * K + 1;
  static constexpr bool Q2 = N1 == 9;
  static constexpr int ax = 1, ay = Q2 ? 9 : N1, az = Q2 ? 89 : N1 * N1;
  static constexpr int bx = Q2 ? 9 : 1, by = Q2 ? 89 : N1, bz = Q2 ? 1 : N1 * N1;
  static constexpr int nx = 1, ny = N1, nz = N1 * N1;
  static constexpr int SA = ax * (N1 - 1) + ay * (N1 - 1) + az * (N1 - 1) + 1;
  static constexpr int SB = bx * (N1 - 1) + by * (N1 - 1) + bz * (N1 - 1) + 1;
  static constexpr int SN = N1 * N1 * N1;
  static constexpr int SS = SA > SB ? (SA > SN ? SA : SN) : (SB > SN ? SB : SN);
  static constexpr int SLOT = SS + ((17 - SS % 16) % 16);   // = 1 mod 16
};
// (the coarse patch region only for TA_CHEB_P01: a smaller footprint lets the
// driver choose a smaller shared-memory carveout, i.e. a larger L1)
template <int K, typename T, int SLOTS, int TM = TA_CHEB_P01>
constexpr size_t gf_smem_bytes() {
  return sizeof(T) * 2 * SLOTS * GfLayout<K>::SLOT +
         (TM == TA_CHEB_P01 ? (size_t)sizeof(T) * SLOTS * GfShape<K>::NCB : 0);
}

// The kernel, register-capped two ways: through the minimum-blocks bound (8 blocks
// of 96 threads, 80 registers; the modes whose working set fits -- plain, X1, 01,
// P01 -- and keep their occupancy), or (_r96) at 96 registers and 7 blocks: TA_CHEB_11
// and TA_CHEB_10 hold g, D^-1 and dv of the epilogue (27 more values) and spill at 80
// (44 bytes; 3.5 % / 2 % slower on c5's finest level).
#define GFAM_NAME gfam_tensor_apply
#define GFAM_ATTR __launch_bounds__(GfBlock<GF_SLOTS>::THREADS, GfBlock<GF_SLOTS>::MIN_BLOCKS)
#include "gfam_kernel.inc"
#undef GFAM_NAME
#undef GFAM_ATTR
#define GFAM_NAME gfam_tensor_apply_r96
#define GFAM_ATTR __maxnreg__(96)
#include "gfam_kernel.inc"
#undef GFAM_NAME
#undef GFAM_ATTR

// 2D form of fam_tensor_apply: a (2k+1)^2 patch has only 2k+1 lines, so one warp
// packs FPW = 32 / (2k+1) families (6 for Q2, 10 for Q1) instead of leaving
// 27 (29) lanes idle.  Lines along x first (gathered into registers), one
// transposition through shared memory, lines along y; interior patch nodes
// stored, the others reduced.
// one warp's work (global warp index gw; s0w, s1w: this warp's FPW x (2k+1)^2 slots)
template <int K, typename T>
__device__ __forceinline__ void fam2d_warp(long gw, T* __restrict__ s0w, T* __restrict__ s1w, int nfam,
                                           const int* __restrict__ xfer, int row, const double* __restrict__ fcoef,
                                           double scale_, const T* __restrict__ x, T* __restrict__ y) {
  constexpr int NP1 = 2 * K + 1, NP = NP1 * NP1, FPW = 32 / NP1;
  const int lane = threadIdx.x & 31;
  const int j = lane / NP1, line = lane % NP1;
  const long f = gw * FPW + j;
  T* const s0j = s0w + (j < FPW ? j : 0) * NP;
  T* const s1j = s1w + (j < FPW ? j : 0) * NP;
  const bool active = j < FPW && f < nfam;
  const int* rp = xfer + (active ? f : 0) * (long)row;
  const T scale = (T)(active && fcoef ? scale_ * __ldg(fcoef + f) : scale_);
  if (active) {        // x lines: line = py, gathered straight into registers
    const int b = line * NP1;
    T u[NP1];
#pragma unroll
    for (int q = 0; q < NP1; ++q) {
      const int gi = decode_dof(__ldg(rp + b + q));
      u[q] = gi >= 0 ? __ldg(x + gi) : T(0);
    }
#pragma unroll
    for (int xx = 0; xx < NP1; ++xx) {
      T a = 0, bb = 0;
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        if (Kt<K>(xx, q) != 0.0) a = fma((T)Kt<K>(xx, q), u[q], a);
        if (Mt<K>(xx, q) != 0.0) bb = fma((T)Mt<K>(xx, q), u[q], bb);
      }
      s0j[b + xx] = a;
      s1j[b + xx] = bb;
    }
  }
  __syncwarp();
  if (active) {        // y lines: line = px
    T a[NP1], bb[NP1];
#pragma unroll
    for (int q = 0; q < NP1; ++q) {
      a[q] = s0j[line + q * NP1];
      bb[q] = s1j[line + q * NP1];
    }
#pragma unroll
    for (int yy = 0; yy < NP1; ++yy) {
      T o = 0;
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        if (Mt<K>(yy, q) != 0.0) o = fma((T)Mt<K>(yy, q), a[q], o);
        if (Kt<K>(yy, q) != 0.0) o = fma((T)Kt<K>(yy, q), bb[q], o);
      }
      const int i = decode_dof(__ldg(rp + line + yy * NP1));
      if (i < 0) continue;
      if (line > 0 && line < 2 * K && yy > 0 && yy < 2 * K) y[i] = scale * o;   // only this family
      else atomicAdd(y + i, scale * o);
    }
  }
}

template <int K, typename T>
__global__ void __launch_bounds__(32 * TENSOR_WARPS)
fam_tensor_apply2d(int nfam, const int* __restrict__ xfer, int row, const double* __restrict__ fcoef,
                   double scale_, const T* __restrict__ x, T* __restrict__ y) {
  constexpr int NP1 = 2 * K + 1, NP = NP1 * NP1, FPW = 32 / NP1;
  __shared__ T s0[TENSOR_WARPS][FPW][NP], s1[TENSOR_WARPS][FPW][NP];
  const int w = threadIdx.x >> 5;
  fam2d_warp<K, T>((long)blockIdx.x * TENSOR_WARPS + w, &s0[w][0][0], &s1[w][0][0], nfam, xfer, row, fcoef, scale_, x,
                   y);
}

// TA_RES in 2D: the V-cycle's residual and restriction d_{l-1} += P^T (d_l - K_l x_l)
// on family patches, warp-packed like fam_tensor_apply2d (x lines gathered, one
// transposition, y lines): r = d|_own - K_f x on each y line, P^T along y in
// registers, one more transposition, P^T along x, (k+1)^2 coarse values added at
// L2 (the same linearity argument as the 3D TA_RES; g is d_l, dc is d_{l-1})
template <int K, typename T>
__global__ void __launch_bounds__(32 * TENSOR_WARPS)
fam_res2d(int nfam, const int* __restrict__ xfer, int row, const double* __restrict__ fcoef, double scale_,
          const T* __restrict__ x, const T* __restrict__ g, T* __restrict__ dc) {
  constexpr int NP1 = 2 * K + 1, NP = NP1 * NP1, FPW = 32 / NP1, N = K + 1;
  __shared__ T s0[TENSOR_WARPS][FPW][NP], s1[TENSOR_WARPS][FPW][NP];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = lane / NP1, line = lane % NP1;
  const long f = ((long)blockIdx.x * TENSOR_WARPS + w) * FPW + j;
  T* const s0j = &s0[w][j < FPW ? j : 0][0];
  T* const s1j = &s1[w][j < FPW ? j : 0][0];
  const bool active = j < FPW && f < nfam;
  const int* rp = xfer + (active ? f : 0) * (long)row;
  const T scale = (T)(active && fcoef ? scale_ * __ldg(fcoef + f) : scale_);
  if (active) {        // x lines: line = py
    const int b = line * NP1;
    T u[NP1];
#pragma unroll
    for (int q = 0; q < NP1; ++q) {
      const int gi = decode_dof(__ldg(rp + b + q));
      u[q] = gi >= 0 ? __ldg(x + gi) : T(0);
    }
#pragma unroll
    for (int xx = 0; xx < NP1; ++xx) {
      T a = 0, bb = 0;
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        if (Kt<K>(xx, q) != 0.0) a = fma((T)Kt<K>(xx, q), u[q], a);
        if (Mt<K>(xx, q) != 0.0) bb = fma((T)Mt<K>(xx, q), u[q], bb);
      }
      s0j[b + xx] = a;
      s1j[b + xx] = bb;
    }
  }
  __syncwarp();
  T rc[N];
#pragma unroll
  for (int c = 0; c < N; ++c) rc[c] = T(0);
  if (active) {        // y lines: line = px; r and P^T along y
    T a[NP1], bb[NP1];
#pragma unroll
    for (int q = 0; q < NP1; ++q) {
      a[q] = s0j[line + q * NP1];
      bb[q] = s1j[line + q * NP1];
    }
#pragma unroll
    for (int yy = 0; yy < NP1; ++yy) {
      T o = 0;
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        if (Mt<K>(yy, q) != 0.0) o = fma((T)Mt<K>(yy, q), a[q], o);
        if (Kt<K>(yy, q) != 0.0) o = fma((T)Kt<K>(yy, q), bb[q], o);
      }
      const int e = __ldg(rp + line + yy * NP1);
      const int i = decode_dof(e);
      if (i < 0) continue;
      const T r = (e >= 0 ? __ldg(g + i) : T(0)) - scale * o;
#pragma unroll
      for (int c = 0; c < N; ++c)
        if (Q<K>::P(yy, c) != 0.0) rc[c] = fma((T)Q<K>::P(yy, c), r, rc[c]);
    }
  }
  __syncwarp();        // every lane has read the y-line inputs
  if (active) {
#pragma unroll
    for (int c = 0; c < N; ++c) s0j[line + NP1 * c] = rc[c];
  }
  __syncwarp();
  if (active && line < N) {   // x lines of the coarse rows: jy = line
    T v[NP1];
#pragma unroll
    for (int q = 0; q < NP1; ++q) v[q] = s0j[q + NP1 * line];
#pragma unroll
    for (int jx = 0; jx < N; ++jx) {
      T acc = T(0);
#pragma unroll
      for (int q = 0; q < NP1; ++q)
        if (Q<K>::P(q, jx) != 0.0) acc = fma((T)Q<K>::P(q, jx), v[q], acc);
      const int ci = __ldg(rp + NP + jx + N * line);
      if (ci >= 0) atomicAdd(dc + ci, acc);
    }
  }
}

// cell_dofs is SoA: dof of local node b of cell c at cell_dofs[b * ldc + c]
template <int D, int K, typename T>
__global__ void __launch_bounds__(128) cell_apply(int n, const int* __restrict__ list,
                                                  const int* __restrict__ cell_dofs, long ldc,
                                                  const double* __restrict__ coef, double scale,
                                                  const T* __restrict__ x, T* __restrict__ y) {
  constexpr int NN = Shape<D, K>::NN;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int c = list ? list[t] : t;
  int idx[NN];
  T u[NN], v[NN];
#pragma unroll
  for (int b = 0; b < NN; ++b) idx[b] = __ldg(cell_dofs + (long)b * ldc + c);
#pragma unroll
  for (int b = 0; b < NN; ++b) u[b] = idx[b] >= 0 ? __ldg(x + idx[b]) : T(0);
  elem_apply<D, K, T>(u, v);
  const T s = (T)(coef ? scale * __ldg(coef + c) : scale);
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

// Levels 0-1 of config 4: cells coarser than the coefficient patches carry an
// explicit element matrix (exact sub-box integration, coef.cpp); y += A_c x_c
// over a cell list (or all cells), thread per (cell, row).
template <int D, int K, typename T>
__global__ void cell_apply_dense(int n, const int* __restrict__ list, const int* __restrict__ cell_dofs, long ldc,
                                 const double* __restrict__ elem, const T* __restrict__ x, T* __restrict__ y) {
  constexpr int NN = Shape<D, K>::NN;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * NN) return;
  const int c = list ? list[t / NN] : t / NN, b = t % NN;
  const int row = cell_dofs[(long)b * ldc + c];
  if (row < 0) return;
  const double* A = elem + ((long)c * NN + b) * NN;
  T s = 0;
  for (int q = 0; q < NN; ++q) {
    const int col = cell_dofs[(long)q * ldc + c];
    if (col >= 0) s = fma((T)A[q], x[col], s);
  }
  atomicAdd(y + row, s);
}
template <int D, int K>
__global__ void cell_diag_dense(int n, const int* __restrict__ cell_dofs, long ldc, const double* __restrict__ elem,
                                double* __restrict__ diag) {
  constexpr int NN = Shape<D, K>::NN;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * NN) return;
  const int c = t / NN, b = t % NN;
  const int row = cell_dofs[(long)b * ldc + c];
  if (row >= 0) atomicAdd(diag + row, elem[((long)c * NN + b) * NN + b]);
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
// Level segments are padded to VEC_PAD doubles with Dinv = g = t = x = 0 in the
// padding, so the grid covers the segment exactly (no bounds branch).
constexpr int VEC_NT = 256;
constexpr int VEC_PAD = 2 * VEC_NT;
// block size of the launches of cheb_step / cheb_range (<= VEC_NT, so that a
// padded segment is a whole number of cheb_step blocks)
#ifndef CHEB_NT_DEFAULT
#define CHEB_NT_DEFAULT 256
#endif
constexpr int CHEB_NT = CHEB_NT_DEFAULT;
static_assert(VEC_PAD % (2 * CHEB_NT) == 0, "cheb_step covers a padded segment exactly");
template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

template <typename S, bool READ_T, bool READ_DV, bool WRITE_DV, bool X_ZERO, bool DV_IS_X = false>
__global__ void __launch_bounds__(VEC_NT) cheb_step(const typename Vec2<S>::type* __restrict__ g,
                                                    const typename Vec2<S>::type* __restrict__ Dinv,
                                                    typename Vec2<S>::type* __restrict__ t,
                                                    typename Vec2<S>::type* __restrict__ dv,
                                                    typename Vec2<S>::type* __restrict__ x, double c1_, double c2_) {
  using V2 = typename Vec2<S>::type;
  const S c1 = (S)c1_, c2 = (S)c2_;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const V2 G = g[i];
  V2 T = {S(0), S(0)}, V = T, X = T;
  if (READ_T) T = t[i];
  const V2 Di = Dinv[i];
  if (!X_ZERO) X = x[i];
  if (READ_DV) V = DV_IS_X ? X : dv[i];
  // reset of the accumulator: the stored zero is made data-dependent on the loaded
  // value so that the store cannot be issued while the load of the same address is
  // in flight (that ordering costs 2.25x on B200: tools/microbench8.cu)
  if (READ_T) t[i] = V2{T.x - T.x, T.y - T.y};
  S dx = c2 * Di.x * (G.x - T.x), dy = c2 * Di.y * (G.y - T.y);
  if (READ_DV) {
    dx = fma(c1, V.x, dx);
    dy = fma(c1, V.y, dy);
  }
  if (WRITE_DV) dv[i] = V2{dx, dy};
  x[i] = V2{X.x + dx, X.y + dy};
}

// The Chebyshev step on [a, n) only (the rows not finished by the fused apply):
// scalar form of cheb_step<T, READ_T = 1, ..., X_ZERO = 0>.
// one row of cheb_range (used by the persistent small-level kernel)
template <typename T, bool READ_DV, bool WRITE_DV, bool DV_IS_X, bool PRO, bool Z1 = false>
__device__ __forceinline__ void cheb_row(long i, const T* __restrict__ g, const T* __restrict__ Dinv, T* __restrict__ t,
                                         T* __restrict__ dv, T* __restrict__ x, double c1_, double c2_, long n_own,
                                         double c0_ = 0) {
  const T G = g[i], Tv = t[i], Di = Dinv[i];
  T X = Z1 ? (T)c0_ * Di * G : x[i];   // Z1: x_1 = c2_0 D^-1 g formed here (0 on ghosts / E rows)
  if (PRO && i < n_own) X = X + dv[i];
  T V = 0;
  if (READ_DV) V = DV_IS_X ? X : dv[i];
  t[i] = Tv - Tv;
  T dd = (T)c2_ * Di * (G - Tv);
  if (READ_DV) dd = fma((T)c1_, V, dd);
  if (WRITE_DV) dv[i] = dd;
  x[i] = X + dd;
}

template <typename T, bool READ_DV, bool WRITE_DV, bool DV_IS_X = false, bool PRO = false, bool Z1 = false>
__global__ void __launch_bounds__(VEC_NT) cheb_range(long a, long n, const T* __restrict__ g,
                                                     const T* __restrict__ Dinv, T* __restrict__ t,
                                                     T* __restrict__ dv, T* __restrict__ x, double c1_, double c2_,
                                                     long n_own = 0, double c0_ = 0) {
  const long i = a + (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T G = g[i], Tv = t[i], Di = Dinv[i];
  T X = Z1 ? (T)c0_ * Di * G : x[i];   // Z1: x_1 = c2_0 D^-1 g (see TA_CHEB_Z1)
  if (PRO && i < n_own) X = X + dv[i];   // x + P x_{l-1} (fam_tensor_apply<TA_CHEB_P01> left it in dv)
  T V = 0;
  if (READ_DV) V = DV_IS_X ? X : dv[i];      // DV_IS_X: dv_0 = x_1 after the first step from 0
  t[i] = Tv - Tv;                       // data-dependent reset (see cheb_step)
  T dd = (T)c2_ * Di * (G - Tv);
  if (READ_DV) dd = fma((T)c1_, V, dd);
  if (WRITE_DV) dv[i] = dd;
  x[i] = X + dd;
}

// x_1 = c0 D^-1 g on the rows in idx (the send rows before a TA_CHEB_Z1 import)
template <typename T>
__global__ void x1_rows(long n, const int* __restrict__ idx, const T* __restrict__ g, const T* __restrict__ Dinv,
                        T* __restrict__ x, double c0) {
  const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) {
    const int i = idx[k];
    x[i] = (T)c0 * Dinv[i] * g[i];
  }
}

// dst[perm[i]] = src[i] (level order -> device order, plan.hpp) and the inverse
__global__ void permute_in(long n, const int* __restrict__ perm, const double* __restrict__ src,
                           double* __restrict__ dst) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[perm[i]] = src[i];
}
__global__ void permute_out(long n, const int* __restrict__ perm, const double* __restrict__ src,
                            double* __restrict__ dst) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

// ------------------------------------------------------------- transfers
// Sum-factorised cell-wise transfers.  Warp per family
// (the 2^d children of one refined level-(l-1) cell, "parent"), persistent
// grid-stride loop.  The family's AoS row xfer[f] = [NP fine patch entries
// (family-patch encoding) | NC coarse DoFs of the parent (-1 Dirichlet)] is
// staged in shared memory, the next family's row is prefetched into registers
// while the current one computes.  With the 1-D embedding P (Q<K>::P, (2k+1) x
// (k+1)) the patch values are P (x) P (x) P applied to the parent's values:
// prolongation runs the three 1-D passes coarse -> fine (x, y, z), restriction
// the transposed passes fine -> coarse (z, y, x).  Each fine node is written
// (prolongation) or summed (restriction) by the one family that owns it, which
// makes both exactly P and P^T (reading R26 of DESIGN.md).
enum : int { XFER_ADD = 0, XFER_SET_E = 1 };
enum : int { RES_PLAIN = 0, RES_VCYCLE = 1, RES_EONLY = 2 };

constexpr int XFER_WARPS = 4;

template <int D, int K>
struct XferShape {
  static constexpr int N = K + 1, NP1 = 2 * K + 1, NC = Shape<D, K>::NN, NP = Shape<D, K>::NP, ROW = NP + NC;
  static constexpr int NR = (ROW + 31) / 32;   // row words per lane
};

template <int D, int K>
__device__ __forceinline__ void row_fetch(const int* __restrict__ xfer, const int* __restrict__ fam_list, int tt,
                                          int lane, int (&r)[XferShape<D, K>::NR]) {
  using S = XferShape<D, K>;
  const int f = fam_list ? __ldg(fam_list + tt) : tt;
  const int* row = xfer + (long)f * S::ROW;
#pragma unroll
  for (int q = 0; q < S::NR; ++q) r[q] = (lane + 32 * q < S::ROW) ? __ldg(row + lane + 32 * q) : -1;
}

template <int D, int K, int MODE, typename T>
__device__ __forceinline__ void warp_prolongate_body(int bid, int nblocks, int* __restrict__ srow, T* __restrict__ b0, T* __restrict__ b1, int nfam, const int* __restrict__ fam_list, const int* __restrict__ xfer,
                const unsigned char* __restrict__ cls_fine, const T* __restrict__ xc, T* __restrict__ xf) {
  using S = XferShape<D, K>;
  constexpr int N = S::N, NP1 = S::NP1, NC = S::NC, NP = S::NP;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = bid * XFER_WARPS + w, GW = nblocks * XFER_WARPS;
  int* const srw = srow + w * S::ROW;
  T* const b0w = b0 + w * NP;
  T* const b1w = b1 + w * NP;
  if (gw >= nfam) return;   // (no block-wide barrier below)
  int nxt[S::NR];
  row_fetch<D, K>(xfer, fam_list, gw, lane, nxt);
  for (int tt = gw; tt < nfam; tt += GW) {
#pragma unroll
    for (int q = 0; q < S::NR; ++q)
      if (lane + 32 * q < S::ROW) srw[lane + 32 * q] = nxt[q];
    __syncwarp();
    if (tt + GW < nfam) row_fetch<D, K>(xfer, fam_list, tt + GW, lane, nxt);
    const int* rw = srw;
    // one memory round trip per family: the parent's values and the owned fine
    // values (read-modify-write below) are requested together, before the passes
    constexpr int NIT = (NP + 31) / 32;
    int vi[NIT];
    T old[NIT];
#pragma unroll
    for (int q = 0; q < NIT; ++q) {
      const int a = lane + 32 * q;
      vi[q] = a < NP ? rw[a] : -1;    // < 0: not owned / Dirichlet
      old[q] = 0;
      if (vi[q] >= 0) {
        if (MODE == XFER_SET_E) old[q] = (cls_fine[vi[q]] & 1) ? T(1) : T(0);
        else old[q] = xf[vi[q]];
      }
    }
    if (lane < NC) {
      const int ci = rw[NP + lane];
      b0w[lane] = ci >= 0 ? __ldg(xc + ci) : T(0);
    }
    __syncwarp();
    T* fine;
    if constexpr (D == 3) {
      // x: c[jz][jy][jx] -> b1[jz][jy][ax];  y: -> b0[jz][ay][ax];  z: -> b1[az][ay][ax]
      xfer_pass<K, true, N * N, 1>(lane, b0w, b1w, N, 1, 0, NP1, 1, 0);
      __syncwarp();
      xfer_pass<K, true, N, NP1>(lane, b1w, b0w, N * NP1, NP1, 1, NP1 * NP1, NP1, 1);
      __syncwarp();
      xfer_pass<K, true, 1, NP1 * NP1>(lane, b0w, b1w, 0, NP1 * NP1, 1, 0, NP1 * NP1, 1);
      fine = b1w;
    } else {
      xfer_pass<K, true, N, 1>(lane, b0w, b1w, N, 1, 0, NP1, 1, 0);
      __syncwarp();
      xfer_pass<K, true, 1, NP1>(lane, b1w, b0w, 0, NP1, 1, 0, NP1, 1);
      fine = b0w;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < NIT; ++q) {
      const int a = lane + 32 * q;
      if (vi[q] < 0) continue;
      if (MODE == XFER_SET_E) {
        if (old[q] != T(0)) xf[vi[q]] = fine[a];
      } else {
        xf[vi[q]] = old[q] + fine[a];
      }
    }
    __syncwarp();
  }
}

template <int D, int K, int MODE, typename T>
__global__ void __launch_bounds__(32 * XFER_WARPS)
warp_prolongate(int nfam, const int* __restrict__ fam_list, const int* __restrict__ xfer,
                const unsigned char* __restrict__ cls_fine, const T* __restrict__ xc, T* __restrict__ xf) {
  using S = XferShape<D, K>;
  __shared__ int srow[XFER_WARPS * S::ROW];
  __shared__ T b0[XFER_WARPS * S::NP], b1[XFER_WARPS * S::NP];
  warp_prolongate_body<D, K, MODE, T>(blockIdx.x, gridDim.x, srow, b0, b1, nfam, fam_list, xfer, cls_fine, xc, xf);
}

template <int D, int K, int MODE, typename T>
__device__ __forceinline__ void warp_restrict_body(int bid, int nblocks, int* __restrict__ srow, T* __restrict__ b0, T* __restrict__ b1, int nfam, const int* __restrict__ fam_list, const int* __restrict__ xfer,
              const unsigned char* __restrict__ cls_fine, const T* __restrict__ v, T* __restrict__ t,
              T* __restrict__ dc) {
  using S = XferShape<D, K>;
  constexpr int N = S::N, NP1 = S::NP1, NC = S::NC, NP = S::NP;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = bid * XFER_WARPS + w, GW = nblocks * XFER_WARPS;
  int* const srw = srow + w * S::ROW;
  T* const b0w = b0 + w * NP;
  T* const b1w = b1 + w * NP;
  if (gw >= nfam) return;   // (no block-wide barrier below)
  int nxt[S::NR];
  row_fetch<D, K>(xfer, fam_list, gw, lane, nxt);
  for (int tt = gw; tt < nfam; tt += GW) {
#pragma unroll
    for (int q = 0; q < S::NR; ++q)
      if (lane + 32 * q < S::ROW) srw[lane + 32 * q] = nxt[q];
    __syncwarp();
    if (tt + GW < nfam) row_fetch<D, K>(xfer, fam_list, tt + GW, lane, nxt);
    const int* rw = srw;
    // residual on the family's owned fine nodes (0 elsewhere); all loads first
    constexpr int NIT = (NP + 31) / 32;
    int ii[NIT];
    T va[NIT], ta[NIT];
#pragma unroll
    for (int q = 0; q < NIT; ++q) {
      const int a = lane + 32 * q;
      ii[q] = a < NP ? rw[a] : -1;
      va[q] = 0;
      ta[q] = 0;
      if (ii[q] >= 0) {
        va[q] = v[ii[q]];
        if (MODE == RES_VCYCLE) ta[q] = t[ii[q]];
        if (MODE == RES_EONLY) ta[q] = (cls_fine[ii[q]] & 1) ? T(0) : T(1);
      }
    }
#pragma unroll
    for (int q = 0; q < NIT; ++q) {
      const int a = lane + 32 * q;
      T r = 0;
      if (ii[q] >= 0) {
        if (MODE == RES_VCYCLE) {
          r = va[q] - ta[q];
          t[ii[q]] = ta[q] - ta[q];             // data-dependent reset (see cheb_step)
        } else if (MODE == RES_EONLY) {
          r = ta[q] == T(0) ? va[q] : T(0);
        } else {
          r = va[q];
        }
      }
      if (a < NP) b0w[a] = r;
    }
    __syncwarp();
    T* coarse;
    if constexpr (D == 3) {
      // z: r[az][ay][ax] -> b1[jz][ay][ax];  y: -> b0[jz][jy][ax];  x: -> b1[jz][jy][jx]
      xfer_pass<K, false, 1, NP1 * NP1>(lane, b0w, b1w, 0, NP1 * NP1, 1, 0, NP1 * NP1, 1);
      __syncwarp();
      xfer_pass<K, false, N, NP1>(lane, b1w, b0w, NP1 * NP1, NP1, 1, N * NP1, NP1, 1);
      __syncwarp();
      xfer_pass<K, false, N * N, 1>(lane, b0w, b1w, NP1, 1, 0, N, 1, 0);
      coarse = b1w;
    } else {
      xfer_pass<K, false, 1, NP1>(lane, b0w, b1w, 0, NP1, 1, 0, NP1, 1);
      __syncwarp();
      xfer_pass<K, false, N, 1>(lane, b1w, b0w, NP1, 1, 0, N, 1, 0);
      coarse = b0w;
    }
    __syncwarp();
    if (lane < NC) {
      const int ci = rw[NP + lane];
      if (ci >= 0) atomicAdd(dc + ci, coarse[lane]);
    }
    __syncwarp();
  }
}

template <int D, int K, int MODE, typename T>
__global__ void __launch_bounds__(32 * XFER_WARPS)
warp_restrict(int nfam, const int* __restrict__ fam_list, const int* __restrict__ xfer,
              const unsigned char* __restrict__ cls_fine, const T* __restrict__ v, T* __restrict__ t,
              T* __restrict__ dc) {
  using S = XferShape<D, K>;
  __shared__ int srow[XFER_WARPS * S::ROW];
  __shared__ T b0[XFER_WARPS * S::NP], b1[XFER_WARPS * S::NP];
  warp_restrict_body<D, K, MODE, T>(blockIdx.x, gridDim.x, srow, b0, b1, nfam, fam_list, xfer, cls_fine, v, t, dc);
}


// ------------------------------------------------------------- small levels in one persistent kernel
// small_vcycle: the whole V(l_s) -- pre-smoothing, residual, restriction on
// levels l_s .. 1, the coarse solve, prolongation and post-smoothing on 1 .. l_s
// -- as ONE cooperative kernel whose phases are separated by grid-wide barriers,
// instead of ~17 launches per level of 2-5 us each (the small levels are launch-
// latency bound).  One rank; levels run by the family-patch kernels (3D tensor
// or 2D), constant coefficient, Cholesky coarse solver.  Every phase is the same
// device body the separate kernels run (fam_tensor_body, fam2d_warp,
// warp_restrict_body, warp_prolongate_body, cheb_row), in the same order as
// vcycle_levels / smooth (device.cu), so results match the launch-per-step cycle.
struct SlkLevel {
  const int* xfer;
  const unsigned char* cls;
  const void* Dinv;        // T*
  long n_fam, n_r1, n_pad, n_owned, off, off_c;
  double scale;
  int row, m, fuse_pro, pad_;
  double c1[16], c2[16];
};
constexpr int SLK_THREADS = 128;

template <int D, int K, typename T>
struct SlkSmem {
  using XS = XferShape<D, K>;
  static constexpr int NP1 = 2 * K + 1, NP2 = NP1 * NP1, FPW2 = 32 / NP1;
  static constexpr size_t tensor = D == 3 ? sizeof(T) * (2 * TensorSmem<K, T>::NS + TensorSmem<K, T>::NCB) : 0;
  static constexpr size_t fam2d = D == 2 ? sizeof(T) * 2 * 4 * FPW2 * NP2 : 0;
  static constexpr size_t xfer = 4 * sizeof(int) * XS::ROW + 2 * 4 * sizeof(T) * XS::NP + 16;
  static constexpr size_t bytes = tensor > fam2d ? (tensor > xfer ? tensor : xfer) : (fam2d > xfer ? fam2d : xfer);
};

// Phase functions of small_vcycle: __noinline__ so that each keeps the register
// budget of its own body (inlining all of them into one kernel exceeds 255
// registers and spills).
template <int D, int K, typename T, int TM>
__device__ __noinline__ void slk_tensor(const SlkLevel* v, unsigned char* smem, T* Dm, T* Xm, T* Tm, T* DVm,
                                        const T* xc, double c1, double c2) {
  T *g = Dm + v->off, *x = Xm + v->off, *t = Tm + v->off, *dv = DVm + v->off;
  if constexpr (D == 3) {
    using TS = TensorSmem<K, T>;
    T* s0 = reinterpret_cast<T*>(smem);
    T* s1 = s0 + TS::NS;
    T* cb = s1 + TS::NS;
    const long nvb = (v->n_fam + TensorCfg<K>::FPB - 1) / TensorCfg<K>::FPB;
    for (long vb = blockIdx.x; vb < nvb; vb += gridDim.x)
      fam_tensor_body<K, T, TM>(vb, s0, s1, cb, (int)v->n_fam, v->xfer, v->row, nullptr, v->scale, x, t, v->n_r1, g,
                                (const T*)v->Dinv, dv, x, c1, c2, xc, 0, nullptr);
  } else {
    constexpr int NP1 = 2 * K + 1, NP = NP1 * NP1, FPW = 32 / NP1;
    const int w = threadIdx.x >> 5;
    T* s0 = reinterpret_cast<T*>(smem) + w * FPW * NP;
    T* s1 = reinterpret_cast<T*>(smem) + (4 + w) * FPW * NP;
    const long nw = (v->n_fam + FPW - 1) / FPW;
    for (long gw = (long)blockIdx.x * 4 + w; gw < nw; gw += (long)gridDim.x * 4)
      fam2d_warp<K, T>(gw, s0, s1, (int)v->n_fam, v->xfer, v->row, nullptr, v->scale, x, t);
  }
}

template <int D, typename T, bool RDV, bool WDV, bool DVX, bool PRO>
__device__ __noinline__ void slk_finish(const SlkLevel* v, T* Dm, T* Xm, T* Tm, T* DVm, double c1, double c2) {
  const long gtid = (long)blockIdx.x * blockDim.x + threadIdx.x, gstride = (long)gridDim.x * blockDim.x;
  const long a = D == 3 ? v->n_r1 : 0;
  for (long i = a + gtid; i < v->n_pad; i += gstride)
    cheb_row<T, RDV, WDV, DVX, PRO>(i, Dm + v->off, (const T*)v->Dinv, Tm + v->off, DVm + v->off, Xm + v->off, c1, c2,
                                    v->n_owned);
}

template <int D, int K, typename T, bool RESTRICT>
__device__ __noinline__ void slk_transfer(const SlkLevel* v, unsigned char* smem, T* Dm, T* Xm, T* Tm) {
  using XS = XferShape<D, K>;
  int* srow = reinterpret_cast<int*>(smem);
  T* b0 = reinterpret_cast<T*>(smem + ((4 * sizeof(int) * XS::ROW + 15) / 16) * 16);
  T* b1 = b0 + 4 * XS::NP;
  if (RESTRICT)
    warp_restrict_body<D, K, RES_VCYCLE, T>(blockIdx.x, gridDim.x, srow, b0, b1, (int)v->n_fam, nullptr, v->xfer, v->cls,
                                            Dm + v->off, Tm + v->off, Dm + v->off_c);
  else
    warp_prolongate_body<D, K, XFER_ADD, T>(blockIdx.x, gridDim.x, srow, b0, b1, (int)v->n_fam, nullptr, v->xfer,
                                            v->cls, Xm + v->off_c, Xm + v->off);
}

template <int D, int K, typename T>
__global__ void __launch_bounds__(SLK_THREADS, 4)
small_vcycle(const SlkLevel* __restrict__ lvs, int ls, T* __restrict__ Dm, T* __restrict__ Xm, T* __restrict__ Tm,
             T* __restrict__ DVm, int nS0, const int* __restrict__ coarse_idx, const double* __restrict__ coarse_inv) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  using SM = SlkSmem<D, K, T>;
  __shared__ __align__(16) unsigned char smem[SM::bytes];
  const long gtid = (long)blockIdx.x * blockDim.x + threadIdx.x, gstride = (long)gridDim.x * blockDim.x;
  // one Chebyshev step: t = K x with the fused epilogue (3D) / t = K x (2D), then
  // the rows the epilogue did not finish
  auto step = [&](const SlkLevel* v, auto tm, auto rdv, auto wdv, auto dvx, auto pro, const T* xc, double c1,
                  double c2) {
    constexpr int TM = decltype(tm)::value;
    if constexpr (D == 3) slk_tensor<D, K, T, TM>(v, smem, Dm, Xm, Tm, DVm, xc, c1, c2);
    else slk_tensor<D, K, T, TA_APPLY>(v, smem, Dm, Xm, Tm, DVm, nullptr, 0.0, 0.0);
    grid.sync();
    slk_finish<D, T, decltype(rdv)::value, decltype(wdv)::value, decltype(dvx)::value, decltype(pro)::value>(
        v, Dm, Xm, Tm, DVm, c1, c2);
    grid.sync();
  };
  using F = std::false_type;
  using Tr = std::true_type;
  using X1 = std::integral_constant<int, TA_CHEB_X1>;
  using C11 = std::integral_constant<int, TA_CHEB_11>;
  using C10 = std::integral_constant<int, TA_CHEB_10>;
  using C01 = std::integral_constant<int, TA_CHEB_01>;
  using C00 = std::integral_constant<int, TA_CHEB_00>;
  using P01 = std::integral_constant<int, TA_CHEB_P01>;
  auto tail_steps = [&](const SlkLevel* v, int j0) {
    for (int j = j0; j < v->m; ++j) {
      if (j == v->m - 1) step(v, C10{}, Tr{}, F{}, F{}, F{}, nullptr, v->c1[j], v->c2[j]);
      else step(v, C11{}, Tr{}, Tr{}, F{}, F{}, nullptr, v->c1[j], v->c2[j]);
    }
  };
  // ---------------- down
  for (int l = ls; l >= 1; --l) {
    const SlkLevel* v = lvs + l;
    T *g = Dm + v->off, *x = Xm + v->off;
    const T* Dv = (const T*)v->Dinv;
    if (v->m > 1) {
      // x_1 = c2_0 D^-1 g (cheb_step<..., X_ZERO>), then the fused steps with dv_0 = x_1
      for (long i = gtid; i < v->n_pad; i += gstride) x[i] = (T)v->c2[0] * Dv[i] * g[i];
      grid.sync();
      step(v, X1{}, Tr{}, Tr{}, Tr{}, F{}, nullptr, v->c1[1], v->c2[1]);
      tail_steps(v, 2);
    } else {
      for (long i = gtid; i < v->n_pad; i += gstride) {
        const T dd = (T)v->c2[0] * Dv[i] * g[i];
        DVm[v->off + i] = dd;
        x[i] = dd;
      }
      grid.sync();
    }
    slk_tensor<D, K, T, TA_APPLY>(v, smem, Dm, Xm, Tm, DVm, nullptr, 0.0, 0.0);   // residual t = K x
    grid.sync();
    slk_transfer<D, K, T, true>(v, smem, Dm, Xm, Tm);                             // d_{l-1} += P^T (d - t)
    grid.sync();
  }
  // ---------------- coarse solve (dense inverse of A_0^S)
  if (blockIdx.x == 0 && nS0 > 0) {
    const T* d0 = Dm + lvs[0].off;
    T* x0 = Xm + lvs[0].off;
    for (int i = threadIdx.x; i < nS0; i += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < nS0; ++j) s = fma(coarse_inv[(long)i * nS0 + j], (double)d0[coarse_idx[j]], s);
      x0[coarse_idx[i]] = (T)s;
    }
  }
  grid.sync();
  // ---------------- up
  for (int l = 1; l <= ls; ++l) {
    const SlkLevel* v = lvs + l;
    if (D == 3 && v->fuse_pro && v->m > 1) {
      step(v, P01{}, F{}, Tr{}, F{}, Tr{}, Xm + v->off_c, 0.0, v->c2[0]);
      tail_steps(v, 1);
    } else {
      slk_transfer<D, K, T, false>(v, smem, Dm, Xm, Tm);                          // x_l += P x_{l-1}
      grid.sync();
      if (v->m == 1) {
        step(v, C00{}, F{}, F{}, F{}, F{}, nullptr, 0.0, v->c2[0]);
      } else {
        step(v, C01{}, F{}, Tr{}, F{}, F{}, nullptr, 0.0, v->c2[0]);
        tail_steps(v, 1);
      }
    }
  }
}

// ------------------------------------------------------------- ghost exchange
// (the wire format is the vector's precision: fp32 ghosts in the mixed-precision V-cycle)
template <typename T>
__global__ void pack(long n, const int* __restrict__ idx, const T* __restrict__ v, T* __restrict__ buf) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = v[idx[i]];
}
// ghosts -> buffer, ghost entries reset (data-dependent, see cheb_step)
template <typename T>
__global__ void pack_zero(long n, const int* __restrict__ idx, T* __restrict__ v, T* __restrict__ buf) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const T a = v[idx[i]];
    buf[i] = a;
    v[idx[i]] = a - a;
  }
}
template <typename T>
__global__ void unpack_set(long n, const int* __restrict__ idx, const T* __restrict__ buf, T* __restrict__ v) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[idx[i]] = buf[i];
}
// an owned DoF may be a ghost of several peers: atomic add
template <typename T>
__global__ void unpack_add(long n, const int* __restrict__ idx, const T* __restrict__ buf, T* __restrict__ v) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(v + idx[i], buf[i]);
}

// ------------------------------------------------------------- misc vector kernels
template <typename T>
__global__ void coarse_solve(int n, const int* __restrict__ sidx, const double* __restrict__ Ainv,
                             const T* __restrict__ d, T* __restrict__ x) {
  int i = threadIdx.x;
  for (; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma(Ainv[(long)i * n + j], (double)d[sidx[j]], s);
    x[sidx[i]] = (T)s;
  }
}

template <typename T>
__global__ void cast_vec(long n, const double* __restrict__ in, T* __restrict__ out) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long stride = (long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = (T)in[i];
}

// MG layout <- leaf order: out[m] = (inv[m] >= 0 ? in[inv[m]] : 0)
// Four consecutive entries per thread: the four index loads are one 16-byte load
// and the four gathers are in flight together (one element per thread and
// iteration left these latency bound).  Callers launch ceil(n / 1024) blocks of
// 256 threads.
template <typename T>
__device__ __forceinline__ void store4(T* p, T a, T b, T c, T d, bool vec) {
  if (vec) {
    if constexpr (sizeof(T) == 8) {
      reinterpret_cast<double2*>(p)[0] = make_double2(a, b);
      reinterpret_cast<double2*>(p)[1] = make_double2(c, d);
    } else {
      *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
    }
  } else {
    p[0] = a; p[1] = b; p[2] = c; p[3] = d;
  }
}

// x1 (optional, [x1_lo, x1_hi) a whole padded level segment, both multiples of 4):
// the first pre-smoothing step from x = 0 on that level, x_1 = c2_0 D^-1 g
// (cheb_step<..., X_ZERO>'s expression), formed here from the values just
// gathered instead of by a pass that re-reads g (the finest level of gmg_vcycle)
template <typename T>
__global__ void __launch_bounds__(256) gather_to_mg(long n, const int* __restrict__ inv, const double* __restrict__ in,
                                                    T* __restrict__ out, long x1_lo = 0, long x1_hi = 0,
                                                    const T* __restrict__ Dinv = nullptr, T* __restrict__ x1 = nullptr,
                                                    double c2_ = 0) {
  const long i0 = ((long)blockIdx.x * 256 + threadIdx.x) * 4;
  const T c2 = (T)c2_;
  if (i0 + 3 < n) {
    const int4 s = *reinterpret_cast<const int4*>(inv + i0);   // inv: device allocation, i0 % 4 == 0
    const bool fx = i0 >= x1_lo && i0 < x1_hi;
    T d0 = T(0), d1 = T(0), d2 = T(0), d3 = T(0);
    if (fx) {
      const T* dp = Dinv + (i0 - x1_lo);
      d0 = __ldg(dp); d1 = __ldg(dp + 1); d2 = __ldg(dp + 2); d3 = __ldg(dp + 3);
    }
    const T a = s.x >= 0 ? (T)__ldg(in + s.x) : T(0), b = s.y >= 0 ? (T)__ldg(in + s.y) : T(0);
    const T c = s.z >= 0 ? (T)__ldg(in + s.z) : T(0), d = s.w >= 0 ? (T)__ldg(in + s.w) : T(0);
    store4(out + i0, a, b, c, d, true);                        // MG layout: device allocation
    if (fx) store4(x1 + i0, c2 * d0 * a, c2 * d1 * b, c2 * d2 * c, c2 * d3 * d, true);
  } else {
    for (long i = i0; i < n; ++i) {
      const int s = inv[i];
      const T a = s >= 0 ? (T)in[s] : T(0);
      out[i] = a;
      if (i >= x1_lo && i < x1_hi) x1[i] = c2 * Dinv[i - x1_lo] * a;
    }
  }
}
// leaf order <- MG layout
template <typename T>
__global__ void __launch_bounds__(256) gather_from_mg(long n, const int* __restrict__ perm, const T* __restrict__ in,
                                                      double* __restrict__ out) {
  const long i0 = ((long)blockIdx.x * 256 + threadIdx.x) * 4;
  if (i0 + 3 < n) {
    const int4 s = *reinterpret_cast<const int4*>(perm + i0);
    const double a = (double)__ldg(in + s.x), b = (double)__ldg(in + s.y);
    const double c = (double)__ldg(in + s.z), d = (double)__ldg(in + s.w);
    store4(out + i0, a, b, c, d, ((unsigned long long)out & 15) == 0);   // out: the caller's leaf vector
  } else {
    for (long i = i0; i < n; ++i) out[i] = (double)in[perm[i]];
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

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

// deterministic final sum of nb partials into *out
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

// z = lam * X ; partial (r, z)   (X: the V-cycle result, fp64 or fp32)
template <typename T>
__global__ void __launch_bounds__(RED_NT) mask_copy_dot(long n, const unsigned char* __restrict__ lam,
                                                        const T* __restrict__ X, const double* __restrict__ r,
                                                        double* __restrict__ z, double* __restrict__ partial) {
  double s = 0.0;
  for (long i = (long)blockIdx.x * RED_NT + threadIdx.x; i < n; i += (long)gridDim.x * RED_NT) {
    double v = lam[i] ? (double)X[i] : 0.0;
    z[i] = v;
    s = fma(r[i], v, s);
  }
  block_store_partial<RED_NT>(s, partial);
}

// beta = sc[2]/sc[0]; p = z + beta p
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
