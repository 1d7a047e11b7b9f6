// sm_100a kernels of the local-smoothing GMG hot path (fp64, no tensor cores:
// the contractions are 3x3 / 5x5 per direction, not a GEMM).
//
//  chunk_apply     fused level operator over chunks of 8 consecutive families:
//                  coalesced R1 load + halo gather into shared memory, family
//                  patch tensor operators (sum factorisation), and the
//                  epilogue on the chunk's own rows: t = Kx, t = g - Kx (residual)
//                  or the Chebyshev-Jacobi step; halo rows reduced
//                  into t with fp64 RED at L2
//  chunk_tail      finishes the reduced rows (R2, R3)
//  cell_apply      same operator over an explicit cell list (leaf cells of the
//                  leaf operator, level 0), thread per cell, atomic scatter
//  cell_diag       diagonal of the level operator
//  cell_load       b += f h^d (w (x) w (x) w) on leaf cells (f = const)
//  cheb_step       Chebyshev-Jacobi vector update over a whole level (first
//                  pre-smoothing step from x = 0), double2 streaming
//  warp_restrict   d_{l-1} += P^T r, warp per family; each
//                  fine node is summed by the one family that owns it
//  warp_prolongate x_l += P x_{l-1} on owned fine nodes (exclusive writes), or
//                  x_l[E] = (P x_{l-1})[E] (hanging / edge values, leaf operator)
//  dot / axpy      CG vector kernels with deterministic two-stage reductions
//
// Family patch table (AoS [n_fam][(2k+1)^d]): v >= 0: level DoF v owned (for
// transfers) by this family; v == -1: Dirichlet node; v <= -2: DoF -2-v owned by
// an earlier family.
#pragma once
#include <cstdint>

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
// Family-patch tensor form of the level operator.  On a family (2^d siblings of
// width h, one coefficient) the sum of the 2^d cell operators is itself a
// Kronecker sum over the (2k+1)^d patch: sum_i (x)_j (j == i ? Kt : Mt) with the
// 1-D matrices Kt, Mt assembled over the two children (P:575-577 applied to the
// patch): 7 one-dimensional passes in 3D, 4 in 2D, ~35% fewer DFMA than the
// 2^d separate cell operators.
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

// One warp applies one family's patch operator: inputs gathered from the
// chunk's shared-memory vector xs through the family's slot table sl
// (LOC_NONE = Dirichlet node, value 0), outputs added to the chunk's
// shared-memory accumulator acc.  Lanes = 1-D lines of the patch; s0/s1 are the
// warp's transposition buffers.
constexpr unsigned short LOC_NONE_D = 0xFFFF;
template <int D, int K>
__device__ __forceinline__ void family_patch_apply(int lane, const unsigned short* __restrict__ sl,
                                                   const double* __restrict__ xs, double* acc, double* s0,
                                                   double* s1, double scale) {
  constexpr int NP1 = 2 * K + 1, NP = Shape<D, K>::NP, NL = NP / NP1;
  if (lane >= NL) return;
  double out[NP1];
  int ob, os;
  if constexpr (D == 3) {
    constexpr int S2 = NP1 * NP1;
    {  // z lines: lane = (px, py)
      double u[NP1];
#pragma unroll
      for (int z = 0; z < NP1; ++z) {
        const unsigned short l = sl[z * S2 + lane];
        u[z] = l != LOC_NONE_D ? xs[l] : 0.0;
      }
#pragma unroll
      for (int z = 0; z < NP1; ++z) {
        double t1 = 0.0, t2 = 0.0;
#pragma unroll
        for (int q = 0; q < NP1; ++q) {
          if (Mt<K>(z, q) != 0.0) t1 = fma(Mt<K>(z, q), u[q], t1);
          if (Kt<K>(z, q) != 0.0) t2 = fma(Kt<K>(z, q), u[q], t2);
        }
        s0[z * S2 + lane] = t1;
        s1[z * S2 + lane] = t2;
      }
    }
    __syncwarp((1u << NL) - 1);
    {  // y lines: lane = (px, pz)
      const int px = lane % NP1, pz = lane / NP1, b = pz * S2 + px;
      double t1[NP1], t2[NP1];
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        t1[q] = s0[b + q * NP1];
        t2[q] = s1[b + q * NP1];
      }
#pragma unroll
      for (int yy = 0; yy < NP1; ++yy) {
        double a = 0.0, bb = 0.0;
#pragma unroll
        for (int q = 0; q < NP1; ++q) {
          if (Mt<K>(yy, q) != 0.0) {
            a = fma(Mt<K>(yy, q), t1[q], a);
            bb = fma(Mt<K>(yy, q), t2[q], bb);
          }
          if (Kt<K>(yy, q) != 0.0) bb = fma(Kt<K>(yy, q), t1[q], bb);
        }
        s0[b + yy * NP1] = a;
        s1[b + yy * NP1] = bb;
      }
    }
    __syncwarp((1u << NL) - 1);
    {  // x lines: lane = (py, pz)
      ob = lane * NP1;
      os = 1;
      double a[NP1], bb[NP1];
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        a[q] = s0[ob + q];
        bb[q] = s1[ob + q];
      }
#pragma unroll
      for (int xx = 0; xx < NP1; ++xx) {
        double o = 0.0;
#pragma unroll
        for (int q = 0; q < NP1; ++q) {
          if (Kt<K>(xx, q) != 0.0) o = fma(Kt<K>(xx, q), a[q], o);
          if (Mt<K>(xx, q) != 0.0) o = fma(Mt<K>(xx, q), bb[q], o);
        }
        out[xx] = scale * o;
      }
    }
  } else {
    {  // x lines: lane = py
      const int b = lane * NP1;
      double u[NP1];
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        const unsigned short l = sl[b + q];
        u[q] = l != LOC_NONE_D ? xs[l] : 0.0;
      }
#pragma unroll
      for (int xx = 0; xx < NP1; ++xx) {
        double a = 0.0, bb = 0.0;
#pragma unroll
        for (int q = 0; q < NP1; ++q) {
          if (Kt<K>(xx, q) != 0.0) a = fma(Kt<K>(xx, q), u[q], a);
          if (Mt<K>(xx, q) != 0.0) bb = fma(Mt<K>(xx, q), u[q], bb);
        }
        s0[b + xx] = a;
        s1[b + xx] = bb;
      }
    }
    __syncwarp((1u << NL) - 1);
    {  // y lines: lane = px
      ob = lane;
      os = NP1;
      double a[NP1], bb[NP1];
#pragma unroll
      for (int q = 0; q < NP1; ++q) {
        a[q] = s0[lane + q * NP1];
        bb[q] = s1[lane + q * NP1];
      }
#pragma unroll
      for (int yy = 0; yy < NP1; ++yy) {
        double o = 0.0;
#pragma unroll
        for (int q = 0; q < NP1; ++q) {
          if (Mt<K>(yy, q) != 0.0) o = fma(Mt<K>(yy, q), a[q], o);
          if (Kt<K>(yy, q) != 0.0) o = fma(Kt<K>(yy, q), bb[q], o);
        }
        out[yy] = scale * o;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NP1; ++q) {
    const unsigned short l = sl[ob + q * os];
    if (l != LOC_NONE_D) atomicAdd(acc + l, out[q]);
  }
}

// ---- async-copy primitives (sm_90+ PTX; TMA bulk engine = UBLKCP in SASS)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (16-byte aligned addresses, size a multiple of 16),
// completion counted in bytes on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Fused level-operator kernel over chunks of CHUNK_F consecutive families
// (device order and tables: plan.hpp).  Persistent CTAs, one warp per family;
// each CTA walks its chunks through a two-stage shared-memory pipeline:
//  * the chunk's R1 rows are one contiguous range: x (and g, D^-1, dv for the
//    epilogue) arrive by TMA bulk copies, the family slot table likewise; the
//    halo x values are gathered with cp.async (8 B) through the halo index list,
//    itself bulk-copied two chunks ahead.  Chunk i+1 streams in while chunk i
//    computes;
//  * every family's patch operator accumulates into shared memory;
//  * R1 rows are complete (no other chunk or rank touches them) and are
//    finished in the epilogue:
//       CM_APPLY  t = K x                     (store)
//       CM_RESID  t = g - K x                 (store; the V-cycle residual)
//       CM_CHEB   dv = c1 dv + c2 D^-1 (g - K x),  x += dv   (Chebyshev-Jacobi step,
//                 P:882-887, x-form of the first-kind recurrence; x updated in place:
//                 R1 values are read only by this CTA)
//    halo rows get their partial sums by fp64 reductions (RED) into t and are
//    finished by chunk_tail (R2, R3 after the ghost export-add).
constexpr int CHUNK_F = 8;
enum : int { CM_APPLY = 0, CM_RESID = 1, CM_CHEB = 2 };

struct ChunkSmem {      // dynamic shared-memory layout (byte offsets), computed on the host
  int acc, s0, s1;      // accumulator, transposition buffers
  int st, stride;       // stage s at st + s * stride: x slots | g | D^-1 | dv | slot table
  int ge, de, ve, sl;   // offsets inside a stage
  int hi, hstride;      // halo index list h at hi + h * hstride
  int mb, total;
};

template <int D, int K>
__host__ __device__ inline ChunkSmem chunk_smem_layout(int max_slots, int max_r1, int max_halo, bool need_g,
                                                       bool need_d, bool need_v) {
  constexpr int NP = Shape<D, K>::NP;
  ChunkSmem L{};
  int o = 0;
  auto take = [&](int bytes) {
    const int r = o;
    o += (bytes + 15) & ~15;
    return r;
  };
  const int ns = max_slots + 2, nr = max_r1 + 2;
  L.acc = take(8 * ns);
  L.s0 = take(8 * CHUNK_F * NP);
  L.s1 = take(8 * CHUNK_F * NP);
  L.st = o;
  take(8 * ns);
  L.ge = need_g ? take(8 * nr) - L.st : 0;
  L.de = need_d ? take(8 * nr) - L.st : 0;
  L.ve = need_v ? take(8 * nr) - L.st : 0;
  L.sl = take(2 * CHUNK_F * NP) - L.st;
  L.stride = o - L.st;
  take(L.stride);
  L.hi = o;
  L.hstride = (4 * (max_halo + 8) + 15) & ~15;
  take(3 * L.hstride);
  L.mb = take(8 * 5);
  L.total = o;
  return L;
}

template <int D, int K, int MODE, bool READ_DV, bool WRITE_DV>
__global__ void __launch_bounds__(32 * CHUNK_F, 2)
chunk_apply(ChunkSmem L, int n_chunks, const int4* __restrict__ meta, const int* __restrict__ halo,
            const unsigned short* __restrict__ loc, int nfam, double scale, double* x, double* __restrict__ t,
            const double* __restrict__ g, const double* __restrict__ Dinv, double* __restrict__ dv, double c1,
            double c2) {
  constexpr int NP = Shape<D, K>::NP, NT = 32 * CHUNK_F;
  constexpr bool NG = MODE != CM_APPLY, ND = MODE == CM_CHEB, NV = MODE == CM_CHEB && READ_DV;
  extern __shared__ __align__(16) unsigned char smem[];
  double* acc = (double*)(smem + L.acc);
  double* s0 = (double*)(smem + L.s0);
  double* s1 = (double*)(smem + L.s1);
  unsigned long long* mb = (unsigned long long*)(smem + L.mb);   // [0,1] stages, [2,3,4] halo lists
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int c0 = blockIdx.x, cs = gridDim.x;
  if (c0 >= n_chunks) return;
  const int my_n = (n_chunks - c0 + cs - 1) / cs;   // chunks of this CTA: c0 + i cs, i < my_n

  // bulk copy of the 16-byte aligned span covering [a, a + n) doubles
  auto span = [](int a, int n, int& a0, int& bytes) {
    a0 = a & ~1;
    bytes = n > 0 ? 8 * (((a + n + 1) & ~1) - a0) : 0;
  };
  auto issue_halo_list = [&](int i) {   // one thread
    const int4 m = __ldg(meta + c0 + i * cs);
    const int h0 = m.z & ~3, hb = m.w > 0 ? 4 * (((m.z + m.w + 3) & ~3) - h0) : 0;
    unsigned long long* b = mb + 2 + i % 3;
    mbar_expect_tx(b, hb);
    if (hb) bulk_g2s(smem + L.hi + (i % 3) * L.hstride, halo + h0, hb, b);
  };
  auto issue_main = [&](int i) {   // bulk part: one thread
    const int c = c0 + i * cs, s = i & 1;
    const int4 m = __ldg(meta + c);
    int a0, bytes;
    span(m.x, m.y, a0, bytes);
    unsigned long long* b = mb + s;
    const unsigned lb = 2 * CHUNK_F * NP;
    mbar_expect_tx(b, lb + bytes * (1 + NG + ND + NV));
    bulk_g2s(smem + L.st + s * L.stride + L.sl, loc + (long)c * CHUNK_F * NP, lb, b);
    if (bytes) {
      bulk_g2s(smem + L.st + s * L.stride, x + a0, bytes, b);
      if (NG) bulk_g2s(smem + L.st + s * L.stride + L.ge, g + a0, bytes, b);
      if (ND) bulk_g2s(smem + L.st + s * L.stride + L.de, Dinv + a0, bytes, b);
      if (NV) bulk_g2s(smem + L.st + s * L.stride + L.ve, dv + a0, bytes, b);
    }
  };
  auto issue_gather = [&](int i) {   // all threads: halo x values, one cp.async group
    const int4 m = __ldg(meta + c0 + i * cs);
    const int* hl = (const int*)(smem + L.hi + (i % 3) * L.hstride) + (m.z & 3);
    double* xh = (double*)(smem + L.st + (i & 1) * L.stride) + m.y + 2;
    for (int j = tid; j < m.w; j += NT) cp_async8(xh + j, x + hl[j]);
    cp_async_commit();
  };

  if (tid == 0) {
    for (int q = 0; q < 5; ++q) mbar_init(mb + q, 1);
    mbar_fence_init();
  }
  for (int i = tid; i < (L.s0 - L.acc) / 8; i += NT) acc[i] = 0.0;
  __syncthreads();
  if (tid == 0) {
    issue_halo_list(0);
    if (my_n > 1) issue_halo_list(1);
    issue_main(0);
  }
  mbar_wait(mb + 2, 0);
  issue_gather(0);

  for (int i = 0; i < my_n; ++i) {
    const int c = c0 + i * cs, s = i & 1;
    // ---- prefetch chunk i+1 (main + halo gather) and the halo list of chunk i+2
    if (i + 1 < my_n) {
      mbar_wait(mb + 2 + (i + 1) % 3, ((i + 1) / 3) & 1);
      if (tid == 0) {
        issue_main(i + 1);
        if (i + 2 < my_n) issue_halo_list(i + 2);
      }
      issue_gather(i + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    mbar_wait(mb + s, (i >> 1) & 1);
    __syncthreads();
    // ---- family patch operators
    const int4 m = __ldg(meta + c);
    const double* xs = (const double*)(smem + L.st + s * L.stride);
    const int f = c * CHUNK_F + w;
    if (f < nfam)
      family_patch_apply<D, K>(lane, (const unsigned short*)(smem + L.st + s * L.stride + L.sl) + w * NP, xs, acc, s0 + w * NP,
                               s1 + w * NP, scale);
    __syncthreads();
    // ---- epilogue: R1 rows finished here, halo rows reduced into t
    const int sh = m.x & 1;
    for (int r = tid; r < m.y; r += NT) {
      const int q = r + sh;
      const long gi = (long)m.x + r;
      const double a = acc[q];
      acc[q] = 0.0;
      if (MODE == CM_APPLY) {
        t[gi] = a;
      } else if (MODE == CM_RESID) {
        t[gi] = ((const double*)(smem + L.st + s * L.stride + L.ge))[q] - a;
      } else {
        double dd = c2 * ((const double*)(smem + L.st + s * L.stride + L.de))[q] * (((const double*)(smem + L.st + s * L.stride + L.ge))[q] - a);
        if (READ_DV) dd = fma(c1, ((const double*)(smem + L.st + s * L.stride + L.ve))[q], dd);
        if (WRITE_DV) dv[gi] = dd;
        x[gi] = xs[q] + dd;
      }
    }
    const int* hl = (const int*)(smem + L.hi + (i % 3) * L.hstride) + (m.z & 3);
    for (int j = tid; j < m.w; j += NT) {
      const int q = m.y + 2 + j;
      atomicAdd(t + hl[j], acc[q]);
      acc[q] = 0.0;
    }
    __syncthreads();
  }
}

// Finishes the rows of [a, a + n) whose operator values were reduced into t
// (R2, R3): CM_RESID t = g - t; CM_CHEB the Chebyshev step with t reset to 0
// (data-dependent zero, see cheb_step).
template <int MODE, bool READ_DV, bool WRITE_DV>
__global__ void __launch_bounds__(256) chunk_tail(long a, long n, const double* __restrict__ g,
                                                  const double* __restrict__ Dinv, double* __restrict__ t,
                                                  double* __restrict__ dv, double* __restrict__ x, double c1,
                                                  double c2) {
  const long i = a + (long)blockIdx.x * 256 + threadIdx.x;
  if (i >= a + n) return;
  const double T = t[i];
  if (MODE == CM_RESID) {
    t[i] = g[i] - T;
  } else {
    t[i] = T - T;
    double dd = c2 * Dinv[i] * (g[i] - T);
    if (READ_DV) dd = fma(c1, dv[i], dd);
    if (WRITE_DV) dv[i] = dd;
    x[i] += dd;
  }
}

// dst[perm[i]] = src[i] (level order -> device order) and the inverse
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
// Level segments are padded to VEC_PAD doubles with Dinv = g = t = x = 0 in the
// padding, so the grid covers the segment exactly (no bounds branch).
constexpr int VEC_NT = 256;
constexpr int VEC_PAD = 2 * VEC_NT;
template <bool READ_T, bool READ_DV, bool WRITE_DV, bool X_ZERO>
__global__ void __launch_bounds__(VEC_NT) cheb_step(const double2* __restrict__ g, const double2* __restrict__ Dinv,
                                                    double2* __restrict__ t, double2* __restrict__ dv,
                                                    double2* __restrict__ x, double c1, double c2) {
  const long i = (long)blockIdx.x * VEC_NT + threadIdx.x;
  const double2 G = g[i];
  double2 T = make_double2(0.0, 0.0), V = T, X = T;
  if (READ_T) T = t[i];
  const double2 Di = Dinv[i];
  if (READ_DV) V = dv[i];
  if (!X_ZERO) X = x[i];
  // reset of the accumulator: the stored zero is made data-dependent on the loaded
  // value so that the store cannot be issued while the load of the same address is
  // in flight (that ordering costs 2.25x on B200: tools/microbench8.cu)
  if (READ_T) t[i] = make_double2(T.x - T.x, T.y - T.y);
  double dx = c2 * Di.x * (G.x - T.x), dy = c2 * Di.y * (G.y - T.y);
  if (READ_DV) {
    dx = fma(c1, V.x, dx);
    dy = fma(c1, V.y, dy);
  }
  if (WRITE_DV) dv[i] = make_double2(dx, dy);
  x[i] = make_double2(X.x + dx, X.y + dy);
}

// ------------------------------------------------------------- transfers
enum : int { XFER_ADD = 0, XFER_SET_E = 1 };
enum : int { RES_PLAIN = 0, RES_T = 1, RES_EONLY = 2 };

constexpr int XFER_NT = 128;
constexpr int XFER_WARPS = 4;

// Warp per family over the AoS transfer table xfer[f] = [NP fine patch entries
// (fam_dofs encoding) | NC coarse DoFs of the parent (-1 Dirichlet)]: one
// contiguous row per family, all indices fetched in one coalesced pass.
template <int D, int K, int MODE>
__global__ void __launch_bounds__(32 * XFER_WARPS)
warp_prolongate(int nfam, const int* __restrict__ fam_list, const int* __restrict__ xfer,
                const unsigned char* __restrict__ cls_fine, const double* __restrict__ xc, double* __restrict__ xf) {
  constexpr int NC = Shape<D, K>::NN, NP = Shape<D, K>::NP, NP1 = 2 * K + 1, N = K + 1, ROW = NP + NC;
  __shared__ double sc[XFER_WARPS][NC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * XFER_WARPS + w;
  if (t >= nfam) return;
  const int f = fam_list ? __ldg(fam_list + t) : t;
  const int* row = xfer + (long)f * ROW;
  constexpr int NIT = (NP + 31) / 32;
  int fine[NIT];
#pragma unroll
  for (int q = 0; q < NIT; ++q) fine[q] = (lane + 32 * q < NP) ? __ldg(row + lane + 32 * q) : -1;
  if (lane < NC) {
    const int ci = __ldg(row + NP + lane);
    sc[w][lane] = ci >= 0 ? __ldg(xc + ci) : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < NIT; ++q) {
    const int a = lane + 32 * q;
    const int v = fine[q];
    if (a >= NP || v < 0) continue;                          // not owned / Dirichlet
    if (MODE == XFER_SET_E && !(cls_fine[v] & 1)) continue;
    double wx[N], wy[N], wz[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      wx[j] = Q<K>::P(a % NP1, j);
      wy[j] = Q<K>::P((a / NP1) % NP1, j);
      wz[j] = D == 3 ? Q<K>::P(a / (NP1 * NP1), j) : 1.0;
    }
    double val = 0.0;
#pragma unroll
    for (int jz = 0; jz < (D == 3 ? N : 1); ++jz)
#pragma unroll
      for (int jy = 0; jy < N; ++jy) {
        double s = 0.0;
#pragma unroll
        for (int jx = 0; jx < N; ++jx) s = fma(wx[jx], sc[w][(jz * N + jy) * N + jx], s);
        val = fma(wy[jy] * wz[jz], s, val);
      }
    if (MODE == XFER_SET_E) xf[v] = val;
    else xf[v] += val;
  }
}

template <int D, int K, int MODE>
__global__ void __launch_bounds__(32 * XFER_WARPS)
warp_restrict(int nfam, const int* __restrict__ fam_list, const int* __restrict__ xfer,
              const unsigned char* __restrict__ cls_fine, const double* __restrict__ v, double* __restrict__ t,
              double* __restrict__ dc) {
  constexpr int NC = Shape<D, K>::NN, NP = Shape<D, K>::NP, NP1 = 2 * K + 1, N = K + 1, ROW = NP + NC;
  __shared__ double sr[XFER_WARPS][NP];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tt = blockIdx.x * XFER_WARPS + w;
  if (tt >= nfam) return;
  const int f = fam_list ? __ldg(fam_list + tt) : tt;
  const int* row = xfer + (long)f * ROW;
  constexpr int NIT = (NP + 31) / 32;
  int fine[NIT];
#pragma unroll
  for (int q = 0; q < NIT; ++q) fine[q] = (lane + 32 * q < NP) ? __ldg(row + lane + 32 * q) : -1;
  const int ci = lane < NC ? __ldg(row + NP + lane) : -1;
  double r[NIT];
#pragma unroll
  for (int q = 0; q < NIT; ++q) {
    const int i = fine[q];
    r[q] = 0.0;
    if (i >= 0) {
      if (MODE == RES_T) {                    // r = t (formed by chunk_apply<CM_RESID>)
        const double tv = t[i];
        r[q] = tv;
        t[i] = tv - tv;                       // data-dependent reset (see cheb_step)
      } else if (MODE == RES_EONLY) {
        r[q] = (cls_fine[i] & 1) ? v[i] : 0.0;
      } else {
        r[q] = v[i];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NIT; ++q)
    if (lane + 32 * q < NP) sr[w][lane + 32 * q] = r[q];
  __syncwarp();
  if (lane < NC && ci >= 0) {
    // fine coordinates with a nonzero weight for coarse node j_d: the coincident
    // node 2 j_d and the odd (mid-edge) nodes 1 (and 3 for K = 2)
    const int j = lane;
    const int jj[3] = {j % N, (j / N) % N, D == 3 ? j / (N * N) : 0};
    double s = 0.0;
#pragma unroll
    for (int qz = 0; qz < (D == 3 ? N : 1); ++qz) {
      const int az = D == 3 ? (qz == 0 ? 2 * jj[2] : 2 * qz - 1) : 0;
      const double wz = D == 3 ? Q<K>::P(az, jj[2]) : 1.0;
#pragma unroll
      for (int qy = 0; qy < N; ++qy) {
        const int ay = qy == 0 ? 2 * jj[1] : 2 * qy - 1;
        const double wyz = wz * Q<K>::P(ay, jj[1]);
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          const int ax = qx == 0 ? 2 * jj[0] : 2 * qx - 1;
          const int a = ax + NP1 * ay + (D == 3 ? NP1 * NP1 * az : 0);
          s = fma(wyz * Q<K>::P(ax, jj[0]), sr[w][a], s);
        }
      }
    }
    atomicAdd(dc + ci, s);
  }
}

// ------------------------------------------------------------- ghost exchange
__global__ void pack(long n, const int* __restrict__ idx, const double* __restrict__ v, double* __restrict__ buf) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = v[idx[i]];
}
// ghosts -> buffer, ghost entries reset (data-dependent, see cheb_step)
__global__ void pack_zero(long n, const int* __restrict__ idx, double* __restrict__ v, double* __restrict__ buf) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double a = v[idx[i]];
    buf[i] = a;
    v[idx[i]] = a - a;
  }
}
__global__ void unpack_set(long n, const int* __restrict__ idx, const double* __restrict__ buf, double* __restrict__ v) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[idx[i]] = buf[i];
}
// an owned DoF may be a ghost of several peers: atomic add
__global__ void unpack_add(long n, const int* __restrict__ idx, const double* __restrict__ buf, double* __restrict__ v) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(v + idx[i], buf[i]);
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
