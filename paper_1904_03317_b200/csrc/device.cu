// Device hierarchy and hot-path driver: V-cycle (local smoothing
// P:413-469), Chebyshev-Jacobi smoother, leaf operator with hanging
// nodes, GMG-preconditioned CG, eigenvalue estimate and coarse
// solve (setup).  One rank per GPU (or per host thread on one GPU in the
// local-ranks test mode); rank-local level vectors = owned DoFs + ghosts with
// one ghost import before and one export-add after every operator that needs
// it.  Every exchange is called by every rank in the same
// order, independently of local sizes.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>

#include "comm.hpp"
#include "device.hpp"
#include "kernels.cuh"
#include "plan.hpp"

namespace gmg {

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) fail(GMG_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

struct DevLevel {
  i64 n = 0, n_owned = 0, n_pad = 0, n_cells = 0, n_fam = 0, n_leaf = 0, n_edge = 0, off = 0;
  int* cell_dofs = nullptr;         // SoA [(k+1)^d][n_cells]
  long ldc = 0;
  double* coef = nullptr;           // config 4, levels >= 2: coefficient per local cell
  double* fcoef = nullptr;          // config 4, levels >= 3: coefficient per local family
  double* elem = nullptr;           // config 4, levels 0-1: [n_cells][nn][nn] element matrices
  unsigned char* cls = nullptr;     // bit0 = E
  double* Dinv = nullptr;           // n_pad entries, 0 on E rows, ghosts and padding
  float* Dinv32 = nullptr;          // the same in fp32 (mixed-precision V-cycle)
  int* fam_dofs = nullptr;          // SoA [(2k+1)^d][n_fam], only for the cell-form family apply (fam_apply)
  int* xfer = nullptr;              // AoS [n_fam][(2k+1)^d + (k+1)^d] fine patch | parent DoFs
  i64 n_r1 = 0;                     // device order (plan.hpp): rows [0, n_r1) finished by the fused apply
  i64 n_gf = 0, n_single = 0;       // grandfamily patches / families left to the family kernel
  int* gx = nullptr;                // [n_gf][GF_ROW] grandfamily tables (plan.hpp)
  int* gr1 = nullptr;               // [n_gf][2] the grandfamily's R1-row run (start, count)
  // several ranks: interior / boundary patch lists (plan.hpp) for the overlap of the
  // ghost import with the interior patches
  int *fam_int = nullptr, *fam_bnd = nullptr, *gf_int = nullptr, *gf_bnd = nullptr;
  i64 n_fam_int = 0, n_fam_bnd = 0, n_gf_int = 0, n_gf_bnd = 0;
  bool split = false;
  cudaEvent_t ev_pack = nullptr, ev_ghost = nullptr;
  int* singles = nullptr;           // families not in a grandfamily
  double* gcoef = nullptr;          // coefficient per grandfamily (config 4)
  bool fuse_pro = false;            // prolongation fused into the first post-smoothing step on EVERY rank
  bool fuse_res = false;            // residual + restriction fused (TA_RES) on EVERY rank
  int* perm = nullptr;              // rank-local level index -> device index (API boundary)
  int* leaf_cells = nullptr;
  int* edge_fams = nullptr;
  double h = 1, scale = 1;          // scale = h^(d-2)
  double lam = 0;
  std::vector<double> c1, c2;
  // exchange plan
  std::vector<int> peers;
  std::vector<i64> send_off, recv_off;
  int* send_idx = nullptr;
  int* recv_idx = nullptr;
  i64 n_send = 0, n_recv = 0;
  i64 nS_global = 0;
  std::vector<double> eig_v;
};

struct DeviceHierarchy {
  int dim = 2, k = 2, L = 0, m = 4;
  double lo = 0.08, hi = 1.2;
  int eig_iters = 10;
  std::vector<DevLevel> lv;
  i64 N = 0, n_leaf = 0, n0_global = 0;
  double *D = nullptr, *X = nullptr, *T = nullptr, *DV = nullptr, *W = nullptr, *Y = nullptr;
  // mixed precision (GMG_MIXED_PRECISION): the V-cycle runs on fp32 copies
  // of the MG-layout buffers; CG and the setup stay fp64
  bool mixed = false;
  bool coarse_cheb = false;     // GMG_COARSE_CHEBYSHEV instead of dense Cholesky
  double coarse_lo = 0, coarse_hi = 0;
  float *D32 = nullptr, *X32 = nullptr, *T32 = nullptr, *DV32 = nullptr;
  double *cx = nullptr, *cr = nullptr, *cp = nullptr, *cq = nullptr, *cz = nullptr;
  double *sbuf = nullptr, *rbuf = nullptr;
  unsigned char* lam_mg = nullptr;
  int* mg_to_leaf = nullptr;        // int32: the MG layout stays below 2^31 entries (checked)
  int* leaf_to_mg = nullptr;
  double* partial = nullptr;
  int nred = 0;
  double* scal = nullptr;       // device scalars
  double* hscal = nullptr;      // pinned host mirror
  int nS0 = 0;                  // level-0 DoFs owned here (all on rank 0)
  double* coarse_inv = nullptr;
  int* coarse_idx = nullptr;
  bool use_graph = true;
  bool tensor_apply = true;     // family-patch tensor apply (GMG_APPLY=cell: per-cell in families)
  int gf_slots = 1;             // grandfamilies per block of gfam_tensor_apply (GMG_GF_SLOTS = 1, 2, 3)
  bool overlap = true;          // several ranks: interior patches overlap the ghost import (GMG_OVERLAP=0: off)
  // small levels 1..slk_ls (+ the coarse solve) run as one persistent kernel (small_vcycle);
  // 0 = off.  Chosen at setup: one rank, family-patch levels, constant coefficient,
  // Cholesky coarse solver, every level 1..slk_ls with <= GMG_SLK_FAM families (2048)
  double z1_c0 = 0;             // c2_0 of the TA_CHEB_Z1 step being launched (x_1 = c2_0 D^-1 g)
  int slk_ls = 0;
  int slk_grid = 0;
  dev::SlkLevel* slk_dev = nullptr;
  cudaStream_t cstream = nullptr;   // the import's side stream
  cudaGraphExec_t vgraph = nullptr;
  // gmg_vcycle's variant: copy_to_mg has already formed the finest level's x_1 =
  // c2_0 D^-1 g (gather_to_mg's x1 arguments), so that level's first pass is skipped
  cudaGraphExec_t vgraph_x1 = nullptr;
  bool skip_x1 = false;             // set while such a V-cycle is launched / captured
  cudaStream_t cap = nullptr;
  long long launches = 0, per_vcycle = 0, per_vcycle_x1 = 0, per_leaf_apply = 0;
  std::vector<std::pair<void*, size_t>> allocs;
  // caller's allocator hooks (gmg_params.dev_alloc / dev_free), else cudaMalloc / cudaFree
  void* (*dev_alloc)(size_t, void*, void*) = nullptr;
  void (*dev_free)(void*, size_t, void*, void*) = nullptr;
  void* alloc_ctx = nullptr;
  int sms = 148;
  std::unique_ptr<Comm> comm;
  // kernel profiler (gmg_profile_vcycle): when set, every launch site of the
  // V-cycle brackets its kernel with two events on the launching stream
  struct ProfRec {
    int kind, level;
    double bytes, bytes_layout;
    cudaEvent_t a, b;
  };
  std::vector<ProfRec>* prof = nullptr;
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  cudaEvent_t ev() {
    if (evnext == evpool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) fail(GMG_E_CUDA, "cudaEventCreate");
      evpool.push_back(e);
    }
    return evpool[evnext++];
  }

  template <class T_>
  T_* alloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    const size_t bytes = n * sizeof(T_);
    if (dev_alloc) {
      p = dev_alloc(bytes, nullptr, alloc_ctx);
      if (!p) fail(GMG_E_OOM, "dev_alloc returned NULL for " + std::to_string(bytes) + " bytes");
    } else {
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e != cudaSuccess) fail(GMG_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    allocs.emplace_back(p, bytes);
    return (T_*)p;
  }
  template <class T_>
  T_* upload(const std::vector<T_>& v) {
    T_* p = alloc<T_>(v.size());
    if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T_), cudaMemcpyHostToDevice));
    return p;
  }
  int vgrid(i64 n, int nt = 256) const {
    i64 b = (n + nt - 1) / nt;
    i64 cap_ = (i64)sms * 16;
    if (b > cap_) b = cap_;
    return (int)(b < 1 ? 1 : b);
  }
};

#define DISPATCH_DK(dim, k, ...)                                   \
  do {                                                             \
    if ((dim) == 2 && (k) == 1) { constexpr int D_ = 2, K_ = 1; __VA_ARGS__; } \
    else if ((dim) == 2 && (k) == 2) { constexpr int D_ = 2, K_ = 2; __VA_ARGS__; } \
    else if ((dim) == 3 && (k) == 1) { constexpr int D_ = 3, K_ = 1; __VA_ARGS__; } \
    else { constexpr int D_ = 3, K_ = 2; __VA_ARGS__; }             \
  } while (0)

// ---------------------------------------------------------------- launch profiler
// One record per bracketed launch: kind (gmg.h GMG_K_*), level, the kernel's
// algorithmic bytes per launch (DESIGN.md §6 definitions) and the bytes of the
// index layout it actually reads.
struct Prof {
  DeviceHierarchy* d;
  cudaStream_t s;
  int kind, level;
  double bytes, layout;
  cudaEvent_t a = nullptr;
  Prof(DeviceHierarchy* d_, cudaStream_t s_, int kind_, int level_, double bytes_, double layout_ = -1)
      : d(d_), s(s_), kind(kind_), level(level_), bytes(bytes_), layout(layout_ < 0 ? bytes_ : layout_) {
    if (d->prof) {
      a = d->ev();
      CK(cudaEventRecord(a, s));
    }
  }
  void end() {
    if (d->prof && a) {
      cudaEvent_t b = d->ev();
      if (cudaEventRecord(b, s) == cudaSuccess) d->prof->push_back({kind, level, bytes, layout, a, b});
    }
    a = nullptr;
  }
  ~Prof() { end(); }
};

// ---------------------------------------------------------------- V-cycle buffers by precision
template <typename T> struct MG;
template <> struct MG<double> {
  static double* D(DeviceHierarchy* d) { return d->D; }
  static double* X(DeviceHierarchy* d) { return d->X; }
  static double* T(DeviceHierarchy* d) { return d->T; }
  static double* DV(DeviceHierarchy* d) { return d->DV; }
  static double* Dinv(DevLevel& v) { return v.Dinv; }
};
template <> struct MG<float> {
  static float* D(DeviceHierarchy* d) { return d->D32; }
  static float* X(DeviceHierarchy* d) { return d->X32; }
  static float* T(DeviceHierarchy* d) { return d->T32; }
  static float* DV(DeviceHierarchy* d) { return d->DV32; }
  static float* Dinv(DevLevel& v) { return v.Dinv32; }
};

// ---------------------------------------------------------------- exchanges
// ghosts <- owners (copy)
template <typename T>
static void import_ghosts(DeviceHierarchy* d, int l, T* vec, cudaStream_t s) {
  if (!d->comm) return;
  DevLevel& v = d->lv[l];
  Prof pr(d, s, GMG_K_EXCHANGE, l, (double)(v.n_send + v.n_recv) * (sizeof(T) + 4 + 8));
  T* sb = reinterpret_cast<T*>(d->sbuf);
  T* rb = reinterpret_cast<T*>(d->rbuf);
  if (v.n_send) {
    dev::pack<T><<<(int)((v.n_send + 255) / 256), 256, 0, s>>>(v.n_send, v.send_idx, vec, sb);
    d->launches++;
  }
  d->comm->exchange(v.peers, sb, v.send_off, rb, v.recv_off, sizeof(T), s);   // wire format = the vector's type
  if (v.n_recv) {
    dev::unpack_set<T><<<(int)((v.n_recv + 255) / 256), 256, 0, s>>>(v.n_recv, v.recv_idx, rb, vec);
    d->launches++;
  }
}
// owners += ghosts; ghosts := 0
template <typename T>
static void export_add(DeviceHierarchy* d, int l, T* vec, cudaStream_t s) {
  if (!d->comm) return;
  DevLevel& v = d->lv[l];
  Prof pr(d, s, GMG_K_EXCHANGE, l, (double)(v.n_send + v.n_recv) * (2 * sizeof(T) + 4 + 8));
  T* sb = reinterpret_cast<T*>(d->sbuf);
  T* rb = reinterpret_cast<T*>(d->rbuf);
  if (v.n_recv) {
    dev::pack_zero<T><<<(int)((v.n_recv + 255) / 256), 256, 0, s>>>(v.n_recv, v.recv_idx, vec, sb);
    d->launches++;
  }
  d->comm->exchange(v.peers, sb, v.recv_off, rb, v.send_off, sizeof(T), s);
  if (v.n_send) {
    dev::unpack_add<T><<<(int)((v.n_send + 255) / 256), 256, 0, s>>>(v.n_send, v.send_idx, rb, vec);
    d->launches++;
  }
}
static void allreduce(DeviceHierarchy* d, double* buf, int n, cudaStream_t s) {
  if (d->comm) d->comm->allreduce(buf, n, s);
}

// ---------------------------------------------------------------- primitives
// grid of the four-entries-per-thread copy kernels (gather_to_mg / gather_from_mg)
static int grid4(i64 n) { return (int)std::max<i64>(1, (n + 1023) / 1024); }

// resident blocks of a fam_tensor_apply instantiation on the whole GPU (the
// prefetch distance of its patch rows)
template <int K, typename T, int TM>
static int tensor_wave(DeviceHierarchy* d) {
  static const int per_sm = [] {
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dev::fam_tensor_apply<K, T, TM>, 32 * dev::TG_WARPS, 0));
    return std::max(nb, 1);
  }();
  return per_sm * d->sms;
}
template <int K>
static int tensor_grid(i64 n_fam) {
  return (int)((n_fam + dev::TensorCfg<K>::FPB - 1) / dev::TensorCfg<K>::FPB);
}

// y += K_l x over a cell list (leaf cells) or, list == nullptr, over all local
// cells.  Full levels >= 1 run family-blocked (y must be zero on entry:
// patch-interior nodes are stored, not added); level 0 and cell lists run
// thread-per-cell.
static int nn_of(const DeviceHierarchy* d) { return d->dim == 3 ? (d->k + 1) * (d->k + 1) * (d->k + 1) : (d->k + 1) * (d->k + 1); }
static int np_of(const DeviceHierarchy* d) {
  return d->dim == 3 ? (2 * d->k + 1) * (2 * d->k + 1) * (2 * d->k + 1) : (2 * d->k + 1) * (2 * d->k + 1);
}
// level operator: x read + y written per level DoF, (k+1)^d index entries
// per cell; layout: the (2k+1)^d patch row per family the tensor kernel reads instead
static double apply_bytes(const DeviceHierarchy* d, const DevLevel& v, size_t vb) {
  return 2.0 * vb * (double)v.n + 4.0 * nn_of(d) * (double)v.n_cells;
}
static double apply_layout(const DeviceHierarchy* d, const DevLevel& v, size_t vb) {
  return 2.0 * vb * (double)v.n + 4.0 * np_of(d) * (double)v.n_fam;
}

// GMG_GF_R96=0: TA_CHEB_11 / TA_CHEB_10 grandfamily kernels at the 80-register cap
// (spilling) instead of gfam_tensor_apply_r96
static bool gf_r96() {
  static const bool on = [] {
    const char* e = std::getenv("GMG_GF_R96");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <int K, typename T, int TM, int SL>
static void launch_gf(DeviceHierarchy* d, DevLevel& v, const T* x, T* y, const T* g, T* dv, T* xw, double c1,
                      double c2, const T* xc, cudaStream_t s, const int* glist = nullptr, i64 ng = -1) {
  using KernelT = decltype(&dev::gfam_tensor_apply<K, T, TM, SL>);
  constexpr bool R96_MODE = (TM == dev::TA_CHEB_11 || TM == dev::TA_CHEB_10) && SL == 1;
  KernelT kern = &dev::gfam_tensor_apply<K, T, TM, SL>;
  if constexpr (R96_MODE) {
    if (gf_r96()) kern = &dev::gfam_tensor_apply_r96<K, T, TM, SL>;
  }
  constexpr size_t smem = dev::gf_smem_bytes<K, T, SL, TM>();
  static const int per_sm = [kern] {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, dev::GfBlock<SL>::THREADS, smem));
    return std::max(nb, 1);
  }();
  static const bool prefetch = [] {
    const char* e = std::getenv("GMG_GF_PREFETCH");
    return !(e && e[0] == '0');
  }();
  // GMG_GF_XPF: 0 off, 1 also prefetch x of the blocks half a wave ahead, 2 and the
  // epilogue's R1-row runs
  static const int xmode = [] {
    const char* e = std::getenv("GMG_GF_XPF");
    return e ? std::atoi(e) : 0;
  }();
  const int wave = per_sm * d->sms;
  if (ng < 0) ng = v.n_gf;
  if (ng == 0) return;
  const int grid = (int)((ng + SL - 1) / SL);
  kern<<<grid, dev::GfBlock<SL>::THREADS, smem, s>>>(
      (int)ng, v.gx, v.gcoef, v.scale, x, y, v.n_r1, g, MG<T>::Dinv(v), dv, xw, c1, c2, xc,
      prefetch ? wave : 0, prefetch && xmode > 0 ? wave / 2 : 0, xmode > 1 ? (const int2*)v.gr1 : nullptr, glist,
      d->z1_c0, v.n_owned);
  d->launches++;
}

// GMG_COL: families per block of the plain operator's column kernel (16 or 32,
// fp32 always 32); 0 (default) = fam_tensor_apply<TA_APPLY>.  Measured slower
// (c3 finest level 283 vs 274 us, DESIGN.md section 6 experiment 13)
static int col_fpc() {
  static const int n = [] {
    const char* e = std::getenv("GMG_COL");
    const int v = e ? std::atoi(e) : 0;
    return v == 0 ? 0 : (v == 32 ? 32 : 16);
  }();
  return n;
}
template <int K, typename T, int FPC>
static void launch_col(DeviceHierarchy* d, DevLevel& v, i64 nf, const int* fl, const T* x, T* y, cudaStream_t s) {
  constexpr size_t smem = dev::col_smem_bytes<K, T, FPC>();
  static const int per_sm = [] {
    CK(cudaFuncSetAttribute(dev::fam_col_apply<K, T, FPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dev::fam_col_apply<K, T, FPC>, dev::ColCfg<K, FPC>::THREADS,
                                                     smem));
    return std::max(nb, 1);
  }();
  const int np = (2 * K + 1) * (2 * K + 1) * (2 * K + 1), nn = (K + 1) * (K + 1) * (K + 1);
  const int grid = (int)((nf + FPC - 1) / FPC);
  dev::fam_col_apply<K, T, FPC><<<grid, dev::ColCfg<K, FPC>::THREADS, smem, s>>>(
      (int)nf, v.xfer, np + nn, v.fcoef, v.scale, x, y, v.n_r1, fl ? 0 : per_sm * d->sms, fl);
  d->launches++;
}

// The 3D tensor operator of one level: grandfamily patches (gfam_tensor_apply)
// plus the remaining families (fam_tensor_apply over the singles list), or all
// families.  Epilogue mode TM, fused Chebyshev arguments as fam_tensor_apply.
// phase: 0 all patches, 1 the interior ones (no ghost node), 2 the boundary ones.
template <int K, typename T, int TM>
static void launch_tensor(DeviceHierarchy* d, DevLevel& v, const T* x, T* y, const T* g, T* dv, T* xw, double c1,
                          double c2, const T* xc, cudaStream_t s, int phase = 0) {
  const int np = (2 * K + 1) * (2 * K + 1) * (2 * K + 1), nn = (K + 1) * (K + 1) * (K + 1);
  if (v.n_gf > 0) {
    const int* gl = phase == 1 ? v.gf_int : (phase == 2 ? v.gf_bnd : nullptr);
    const i64 ng = phase == 1 ? v.n_gf_int : (phase == 2 ? v.n_gf_bnd : v.n_gf);
    if (d->gf_slots == 1) launch_gf<K, T, TM, 1>(d, v, x, y, g, dv, xw, c1, c2, xc, s, gl, ng);
    else if (d->gf_slots == 2) launch_gf<K, T, TM, 2>(d, v, x, y, g, dv, xw, c1, c2, xc, s, gl, ng);
    else launch_gf<K, T, TM, 3>(d, v, x, y, g, dv, xw, c1, c2, xc, s, gl, ng);
  }
  const int* fl = phase == 1 ? v.fam_int : (phase == 2 ? v.fam_bnd : (v.n_gf > 0 ? v.singles : nullptr));
  const i64 nf = phase == 1 ? v.n_fam_int : (phase == 2 ? v.n_fam_bnd : (v.n_gf > 0 ? v.n_single : v.n_fam));
  if (nf > 0) {
    if constexpr (TM == dev::TA_APPLY) {
      if (col_fpc() > 0) {   // the plain operator: column kernel (fam_col_apply)
        if (col_fpc() == 16 && sizeof(T) == 8) launch_col<K, T, 16>(d, v, nf, fl, x, y, s);
        else launch_col<K, T, 32>(d, v, nf, fl, x, y, s);
        return;
      }
    }
    if constexpr (K == 2)
      dev::fam_tensor_apply<K, T, TM><<<tensor_grid<K>(nf), 32 * dev::TG_WARPS, 0, s>>>(
          (int)nf, v.xfer, np + nn, v.fcoef, v.scale, x, y, v.n_r1, g, MG<T>::Dinv(v), dv, xw, c1, c2, xc,
          fl ? 0 : tensor_wave<K, T, TM>(d), fl, d->z1_c0, v.n_owned);
    else
      dev::fam_tensor_apply<K, T, TM><<<tensor_grid<K>(nf), 32 * dev::TG_WARPS, 0, s>>>(
          (int)nf, v.xfer, np + nn, v.fcoef, v.scale, x, y, v.n_r1, g, MG<T>::Dinv(v), dv, xw, c1, c2, xc, 0, fl,
          d->z1_c0, v.n_owned);
    d->launches++;
  }
}

// ghost import of x followed by the tensor operator on level l: with several
// ranks and a split level, the import runs on the side stream while the interior
// patches (no ghost node) compute, the boundary patches after it
template <int K, typename T, int TM>
static void import_and_tensor(DeviceHierarchy* d, int l, T* x, T* y, const T* g, T* dv, T* xw, double c1, double c2,
                              const T* xc, cudaStream_t s) {
  DevLevel& v = d->lv[l];
  if (!(d->comm && d->overlap && v.split)) {
    import_ghosts(d, l, x, s);
    launch_tensor<K, T, TM>(d, v, x, y, g, dv, xw, c1, c2, xc, s);
    return;
  }
  CK(cudaEventRecord(v.ev_pack, s));
  CK(cudaStreamWaitEvent(d->cstream, v.ev_pack, 0));
  import_ghosts(d, l, x, d->cstream);
  CK(cudaEventRecord(v.ev_ghost, d->cstream));
  launch_tensor<K, T, TM>(d, v, x, y, g, dv, xw, c1, c2, xc, s, 1);
  CK(cudaStreamWaitEvent(s, v.ev_ghost, 0));
  launch_tensor<K, T, TM>(d, v, x, y, g, dv, xw, c1, c2, xc, s, 2);
}

template <typename T>
static void k_apply(DeviceHierarchy* d, int l, const int* list, i64 n, const T* x, T* y, cudaStream_t s) {
  if (n == 0) return;
  DevLevel& v = d->lv[l];
  const bool full = list == nullptr && l > 0 && v.n_fam > 0;
  Prof pr(d, s, full || list == nullptr ? GMG_K_APPLY : GMG_K_LEAF_APPLY, l,
          list == nullptr ? apply_bytes(d, v, sizeof(T)) : (2.0 * sizeof(T) + 4.0) * nn_of(d) * (double)n,
          list == nullptr && full ? apply_layout(d, v, sizeof(T)) : -1.0);
  if (v.elem) {                                   // config 4, levels 0-1: explicit element matrices
    const int nt = 128;
    const int nn = d->dim == 3 ? (d->k + 1) * (d->k + 1) * (d->k + 1) : (d->k + 1) * (d->k + 1);
    DISPATCH_DK(d->dim, d->k, (dev::cell_apply_dense<D_, K_, T><<<(int)((n * nn + nt - 1) / nt), nt, 0, s>>>(
                                  (int)n, list, v.cell_dofs, v.ldc, v.elem, x, y)));
  } else if (full && (v.coef == nullptr || v.fcoef != nullptr) && d->tensor_apply) {
    const int np = d->dim == 3 ? (2 * d->k + 1) * (2 * d->k + 1) * (2 * d->k + 1) : (2 * d->k + 1) * (2 * d->k + 1);
    const int nn = d->dim == 3 ? (d->k + 1) * (d->k + 1) * (d->k + 1) : (d->k + 1) * (d->k + 1);
    if (d->dim == 2) {   // several families per warp (fam_tensor_apply2d)
      const int fpw = 32 / (2 * d->k + 1), per_block = fpw * dev::TENSOR_WARPS;
      const int grid = (int)((v.n_fam + per_block - 1) / per_block);
      if (d->k == 2)
        dev::fam_tensor_apply2d<2, T><<<grid, 32 * dev::TENSOR_WARPS, 0, s>>>((int)v.n_fam, v.xfer, np + nn,
                                                                               v.fcoef, v.scale, x, y);
      else
        dev::fam_tensor_apply2d<1, T><<<grid, 32 * dev::TENSOR_WARPS, 0, s>>>((int)v.n_fam, v.xfer, np + nn,
                                                                               v.fcoef, v.scale, x, y);
    } else {
      if (d->k == 2)
        launch_tensor<2, T, dev::TA_APPLY>(d, v, x, y, nullptr, nullptr, nullptr, 0.0, 0.0, nullptr, s);
      else
        launch_tensor<1, T, dev::TA_APPLY>(d, v, x, y, nullptr, nullptr, nullptr, 0.0, 0.0, nullptr, s);
      d->launches--;     // counted per kernel in launch_tensor
    }
  } else if (full) {                              // per-cell coefficients inside a family (config 4, level 2)
    DISPATCH_DK(d->dim, d->k, {
      constexpr int FPB = dev::FamCfg<D_, K_>::FPB;
      int grid = (int)((v.n_fam + FPB - 1) / FPB);
      dev::fam_apply<D_, K_, T><<<grid, FPB * (1 << D_), 0, s>>>((int)v.n_fam, v.fam_dofs, v.coef, v.scale, x, y);
    });
  } else {
    const int nt = 128;
    int grid = (int)((n + nt - 1) / nt);
    DISPATCH_DK(d->dim, d->k, (dev::cell_apply<D_, K_, T><<<grid, nt, 0, s>>>((int)n, list, v.cell_dofs, v.ldc, v.coef,
                                                                              v.scale, x, y)));
  }
  d->launches++;
}

// t = K_l x on owned rows: ghost import of x, local family apply, export-add of t
template <typename T>
static void apply_full(DeviceHierarchy* d, int l, T* x, T* t, cudaStream_t s) {
  DevLevel& v = d->lv[l];
  if (d->comm && d->overlap && v.split) {        // 3D tensor level split into interior / boundary patches
    Prof pr(d, s, GMG_K_APPLY, l, apply_bytes(d, v, sizeof(T)), apply_layout(d, v, sizeof(T)));
    if (d->k == 2)
      import_and_tensor<2, T, dev::TA_APPLY>(d, l, x, t, nullptr, nullptr, nullptr, 0.0, 0.0, nullptr, s);
    else
      import_and_tensor<1, T, dev::TA_APPLY>(d, l, x, t, nullptr, nullptr, nullptr, 0.0, 0.0, nullptr, s);
  } else {
    import_ghosts(d, l, x, s);
    k_apply(d, l, nullptr, v.n_cells, x, t, s);
  }
  export_add(d, l, t, s);
}

// The transfer kernels are persistent (grid-stride over families): launch one
// resident wave, not more -- with a second partial wave the late blocks hold the
// same share of families and finish a third of a block's time after the rest.
template <typename Kern>
static int xfer_grid(DeviceHierarchy* d, i64 nf, Kern kern) {
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * dev::XFER_WARPS, 0));
  return (int)std::max<i64>(1, std::min<i64>((nf + dev::XFER_WARPS - 1) / dev::XFER_WARPS,
                                             (i64)std::max(per_sm, 1) * d->sms));
}

template <int MODE, typename T>
static void k_restrict(DeviceHierarchy* d, int l, const int* list, i64 nf, const T* vin, T* t, T* dc,
                       cudaStream_t s) {
  if (nf == 0) return;
  DevLevel& f = d->lv[l];
  // r = d - t read (two vectors, MODE RES_VCYCLE; one otherwise) and t reset per fine
  // row, the family's xfer row, d_{l-1} read-modify-written per coarse row
  const double fine_vecs = MODE == dev::RES_VCYCLE ? 3.0 : 1.0;
  Prof pr(d, s, list ? GMG_K_OTHER : GMG_K_RESTRICT, l,
          list ? 0.0 : fine_vecs * sizeof(T) * (double)f.n + 4.0 * (np_of(d) + nn_of(d)) * (double)nf +
                        2.0 * sizeof(T) * (double)d->lv[l - 1].n);
  DISPATCH_DK(d->dim, d->k, (dev::warp_restrict<D_, K_, MODE, T><<<xfer_grid(d, nf, dev::warp_restrict<D_, K_, MODE, T>), 32 * dev::XFER_WARPS, 0, s>>>(
                                (int)nf, list, f.xfer, f.cls, vin, t, dc)));
  d->launches++;
}

template <int MODE, typename T>
static void k_prolongate(DeviceHierarchy* d, int l, const int* list, i64 nf, const T* xc, T* xf,
                         cudaStream_t s) {
  if (nf == 0) return;
  DevLevel& f = d->lv[l];
  Prof pr(d, s, list ? GMG_K_OTHER : GMG_K_PROLONGATE, l,
          list ? 0.0 : 2.0 * sizeof(T) * (double)f.n + 4.0 * (np_of(d) + nn_of(d)) * (double)nf +
                        sizeof(T) * (double)d->lv[l - 1].n);
  DISPATCH_DK(d->dim, d->k, (dev::warp_prolongate<D_, K_, MODE, T><<<xfer_grid(d, nf, dev::warp_prolongate<D_, K_, MODE, T>), 32 * dev::XFER_WARPS, 0, s>>>(
                                (int)nf, list, f.xfer, f.cls, xc, xf)));
  d->launches++;
}

template <typename T, bool RT, bool RDV, bool WDV, bool XZ, bool DVX = false>
static void k_cheb(DeviceHierarchy* d, DevLevel& v, const T* g, T* t, T* dv, T* x, double c1, double c2,
                   cudaStream_t s) {
  if (v.n_pad == 0) return;
  using V2 = typename dev::Vec2<T>::type;
  // per padded row: g, D^-1 (+ t, dv, x) read; x (+ dv, t) written
  const int nvec = 3 + (RT ? 2 : 0) + (RDV && !DVX ? 1 : 0) + (!XZ ? 1 : 0) + (WDV ? 1 : 0);
  Prof pr(d, s, GMG_K_CHEB_STREAM_FULL, (int)(&v - d->lv.data()), (double)nvec * sizeof(T) * (double)v.n_pad);
  // n_pad is a multiple of VEC_PAD: the grid covers the padded segment exactly
  dev::cheb_step<T, RT, RDV, WDV, XZ, DVX><<<(int)(v.n_pad / (2 * dev::CHEB_NT)), dev::CHEB_NT, 0, s>>>(
      (const V2*)g, (const V2*)MG<T>::Dinv(v), (V2*)t, (V2*)dv, (V2*)x, c1, c2);
  d->launches++;
}

// One Chebyshev step j >= 1 (or the first from a nonzero x): t = K x with the
// rows of R1 finished inside the operator kernel (fam_tensor_apply<TM>), the rest
// by the streaming pass over [n_r1, n_pad).  Falls back to operator + full-level
// streaming step where the level has no R1 (2D, coefficient levels, level 0).
template <typename T, int TM, bool RDV, bool WDV, bool DVX = false>
static void cheb_step_fused(DeviceHierarchy* d, int l, const T* g, T* x, T* t, T* dv, double c1, double c2,
                            cudaStream_t s, const T* xc = nullptr, double c0 = 0.0) {
  constexpr bool PRO = TM == dev::TA_CHEB_P01;   // x + P x_{l-1} (xc) fused in; only called where n_r1 > 0
  constexpr bool Z1 = TM == dev::TA_CHEB_Z1;     // x_1 = c0 D^-1 g formed in the kernels; only where n_r1 > 0
  DevLevel& v = d->lv[l];
  if (Z1) {
    if (v.n_r1 == 0) throw Error(GMG_E_STATE, "TA_CHEB_Z1 on a level without R1");
    d->z1_c0 = c0;
    if (d->comm && v.n_send) {   // the owners' send rows carry x_1 for the ghost import
      dev::x1_rows<T><<<(int)((v.n_send + 255) / 256), 256, 0, s>>>(v.n_send, v.send_idx, g, MG<T>::Dinv(v), x, c0);
      d->launches++;
    }
  }
  if (v.n_r1 > 0) {
    const int np = (2 * d->k + 1) * (2 * d->k + 1) * (2 * d->k + 1), nn = (d->k + 1) * (d->k + 1) * (d->k + 1);
    // the operator's x gather and index rows, t (reduced) on the rows outside R1,
    // and on the R1 rows the Chebyshev vectors: g, D^-1 (+ dv) read, x (+ dv) written
    const double vb = sizeof(T);
    const int r1v = 3 + (RDV && !DVX ? 1 : 0) + (WDV ? 1 : 0);
    double fb = vb * (double)v.n + vb * (double)(v.n - v.n_r1) + r1v * vb * (double)v.n_r1;
    if (PRO) fb += vb * (double)d->lv[l - 1].n + vb * (double)(v.n_owned - v.n_r1);
    const double idx = 4.0 * nn * (double)v.n_cells + (PRO ? 4.0 * nn * (double)v.n_fam : 0.0);
    const double idx_layout = 4.0 * np * (double)v.n_fam + (PRO ? 4.0 * nn * (double)v.n_fam : 0.0);
    const int kind = (TM == dev::TA_CHEB_X1 || Z1) ? GMG_K_CHEB_X1 : TM == dev::TA_CHEB_11 ? GMG_K_CHEB_11
                   : TM == dev::TA_CHEB_10 ? GMG_K_CHEB_10 : TM == dev::TA_CHEB_P01 ? GMG_K_CHEB_P01
                   : TM == dev::TA_CHEB_01 ? GMG_K_CHEB_01 : GMG_K_CHEB_00;
    Prof pr(d, s, kind, l, fb + idx, fb + idx_layout);
    if (d->k == 2)
      import_and_tensor<2, T, TM>(d, l, x, t, g, dv, x, c1, c2, xc, s);
    else
      import_and_tensor<1, T, TM>(d, l, x, t, g, dv, x, c1, c2, xc, s);
    pr.end();
    export_add(d, l, t, s);
    const i64 n = v.n_pad - v.n_r1;
    if (n > 0) {
      const int nvec = 6 + (RDV && !DVX ? 1 : 0) + (WDV ? 1 : 0) + (PRO ? 1 : 0);   // g D t x (+dv) | t x (+dv)
      Prof pr2(d, s, GMG_K_CHEB_STREAM, l, (double)nvec * sizeof(T) * (double)n);
      dev::cheb_range<T, RDV, WDV, DVX, PRO, Z1><<<(int)((n + dev::CHEB_NT - 1) / dev::CHEB_NT), dev::CHEB_NT, 0, s>>>(
          v.n_r1, v.n_pad, g, MG<T>::Dinv(v), t, dv, x, c1, c2, v.n_owned, c0);
      d->launches++;
    }
    d->z1_c0 = 0;
  } else {
    if (PRO) throw Error(GMG_E_STATE, "fused prolongation on a level without R1");
    import_ghosts(d, l, x, s);
    k_apply(d, l, nullptr, v.n_cells, (const T*)x, t, s);
    export_add(d, l, t, s);
    k_cheb<T, true, RDV, WDV, false, DVX>(d, v, g, t, dv, x, c1, c2, s);
  }
}

// GMG_Z1=1: TA_CHEB_Z1 instead of the pass x_1 = c2_0 D^-1 g followed by TA_CHEB_X1.
// Off by default: the doubled gather (D^-1 and g at every patch node) slows the
// step-1 kernels by about what the saved pass costs (c5 19.24 vs 19.34 ms, c3 7.58
// vs 7.55 ms)
static bool z1_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GMG_Z1");
    return e && e[0] == '1';
  }();
  return on;
}

// Chebyshev-Jacobi smoothing on level l with rhs g, state x (x-form of the
// first-kind recurrence: r_j = D^-1 (g - K x_j), dv_j = c1_j dv_{j-1} + c2_j r_j,
// x_{j+1} = x_j + dv_j; D^-1 = 0 on E rows and ghosts keeps those entries fixed).
template <typename T>
static void smooth(DeviceHierarchy* d, int l, const T* g, T* x, T* t, T* dv, bool x_zero, cudaStream_t s,
                   const T* xc = nullptr) {
  DevLevel& v = d->lv[l];
  const int m = (int)v.c1.size();     // degree d->m on levels >= 1, the coarse degree on level 0
  if (m == 0) return;
  int j0 = 1;
  if (xc) {                            // post-smoothing with x + P x_{l-1} fused into step 0 (prolong_fusable)
    cheb_step_fused<T, dev::TA_CHEB_P01, false, true>(d, l, g, x, t, dv, 0.0, v.c2[0], s, xc);
  } else if (x_zero && m > 1 && v.n_r1 > 0 && z1_enabled()) {
    // x_1 = dv_0 = c2_0 D^-1 g is formed inside the step-1 kernels (TA_CHEB_Z1): no pass for it
    cheb_step_fused<T, dev::TA_CHEB_Z1, true, true, true>(d, l, g, x, t, dv, v.c1[1], v.c2[1], s, nullptr, v.c2[0]);
    j0 = 2;
  } else if (x_zero && m > 1) {
    // x_1 = dv_0 = c2_0 D^-1 g: only x is stored, the next step reads dv_0 from x
    if (!(d->skip_x1 && l == d->L)) k_cheb<T, false, false, false, true>(d, v, g, t, dv, x, 0.0, v.c2[0], s);
    cheb_step_fused<T, dev::TA_CHEB_X1, true, true, true>(d, l, g, x, t, dv, v.c1[1], v.c2[1], s);
    j0 = 2;
  } else if (x_zero) {
    k_cheb<T, false, false, true, true>(d, v, g, t, dv, x, 0.0, v.c2[0], s);
  } else if (m == 1) {
    cheb_step_fused<T, dev::TA_CHEB_00, false, false>(d, l, g, x, t, dv, 0.0, v.c2[0], s);
  } else {
    cheb_step_fused<T, dev::TA_CHEB_01, false, true>(d, l, g, x, t, dv, 0.0, v.c2[0], s);
  }
  for (int j = j0; j < m; ++j) {
    if (j == m - 1) cheb_step_fused<T, dev::TA_CHEB_10, true, false>(d, l, g, x, t, dv, v.c1[j], v.c2[j], s);
    else cheb_step_fused<T, dev::TA_CHEB_11, true, true>(d, l, g, x, t, dv, v.c1[j], v.c2[j], s);
  }
}

template <typename T>
static void coarse(DeviceHierarchy* d, T* d0, T* x0, T* t0, T* dv0, cudaStream_t s) {
  if (d->coarse_cheb) {                 // collective: every rank joins the level-0 exchanges
    smooth(d, 0, d0, x0, t0, dv0, true, s);
    return;
  }
  if (d->nS0 == 0) return;
  Prof pr(d, s, GMG_K_COARSE, 0, (double)d->nS0 * d->nS0 * 8.0);
  dev::coarse_solve<T><<<1, 256, 0, s>>>(d->nS0, d->coarse_idx, d->coarse_inv, d0, x0);
  d->launches++;
}

// The prolongation can ride on the first post-smoothing step where that step runs
// the fused operator kernel (R1 present, degree >= 2; GMG_FUSE_PROLONG=0 turns
// it off for comparison).  The decision is collective (fuse_pro, set at setup):
// the fused path imports x_l before adding P x_{l-1} (every rank adds it to its
// ghosts itself), the separate path after, so ranks choosing differently would
// exchange inconsistent ghost values.
static bool prolong_fusable(DeviceHierarchy* d, int l) {
  static const bool on = [] {
    const char* e = std::getenv("GMG_FUSE_PROLONG");
    return !(e && e[0] == '0');
  }();
  return on && d->lv[l].fuse_pro && d->lv[l].c1.size() > 1;
}

// The V-cycle's residual and restriction as one operator pass (kernels.cuh TA_RES):
// d_{l-1} += P^T (d_l - K_l x_l) with every family / grandfamily patch restricting
// its own contribution, on the levels the tensor kernels run, 3D and 2D (GMG_FUSE_RES=0:
// plain operator + export-add of t + warp_restrict).  The decision is collective
// (fuse_res, set at setup): the level's t is neither written nor export-added,
// so ranks choosing differently would mismatch their exchanges; d_{l-1} is
// export-added by the caller as before.
static bool res_fusable(DeviceHierarchy* d, int l) {
  static const bool on = [] {
    const char* e = std::getenv("GMG_FUSE_RES");
    return !(e && e[0] == '0');
  }();
  return on && d->lv[l].fuse_res;
}
template <typename T>
static void res_restrict(DeviceHierarchy* d, int l, T* x, const T* g, T* gc, cudaStream_t s) {
  DevLevel& v = d->lv[l];
  // x gathered and d read per level DoF, the operator's index per cell, the parents'
  // (k+1)^d coarse DoFs per family, d_{l-1} read-modify-written per coarse row
  const double vb = sizeof(T), coarse = 2.0 * vb * (double)d->lv[l - 1].n + 4.0 * nn_of(d) * (double)v.n_fam;
  Prof pr(d, s, GMG_K_RES_RESTRICT, l, 2.0 * vb * (double)v.n + 4.0 * nn_of(d) * (double)v.n_cells + coarse,
          2.0 * vb * (double)v.n + 4.0 * np_of(d) * (double)v.n_fam + coarse);
  if (d->dim == 2) {           // warp-packed families (fam_res2d)
    import_ghosts(d, l, x, s);
    if (v.n_fam == 0) return;
    const int np = (2 * d->k + 1) * (2 * d->k + 1), nn = (d->k + 1) * (d->k + 1);
    const int fpw = 32 / (2 * d->k + 1), per_block = fpw * dev::TENSOR_WARPS;
    const int grid = (int)((v.n_fam + per_block - 1) / per_block);
    if (d->k == 2)
      dev::fam_res2d<2, T><<<grid, 32 * dev::TENSOR_WARPS, 0, s>>>((int)v.n_fam, v.xfer, np + nn, v.fcoef, v.scale,
                                                                    x, g, gc);
    else
      dev::fam_res2d<1, T><<<grid, 32 * dev::TENSOR_WARPS, 0, s>>>((int)v.n_fam, v.xfer, np + nn, v.fcoef, v.scale,
                                                                    x, g, gc);
    d->launches++;
  } else if (d->k == 2) {
    import_and_tensor<2, T, dev::TA_RES>(d, l, x, gc, g, nullptr, nullptr, 0.0, 0.0, nullptr, s);
  } else {
    import_and_tensor<1, T, dev::TA_RES>(d, l, x, gc, g, nullptr, nullptr, 0.0, 0.0, nullptr, s);
  }
}

// V(slk_ls) in one cooperative kernel (kernels.cuh small_vcycle)
template <typename T>
static void run_small_levels(DeviceHierarchy* d, cudaStream_t s) {
  T *D = MG<T>::D(d), *X = MG<T>::X(d), *Tb = MG<T>::T(d), *DV = MG<T>::DV(d);
  int ls = d->slk_ls, nS0 = d->nS0;
  const int* cidx = d->coarse_idx;
  const double* cinv = d->coarse_inv;
  const dev::SlkLevel* lv = d->slk_dev;
  void* args[] = {(void*)&lv, (void*)&ls, (void*)&D, (void*)&X, (void*)&Tb, (void*)&DV, (void*)&nS0, (void*)&cidx,
                  (void*)&cinv};
  Prof pr(d, s, GMG_K_SMALL, ls, 0.0);
  void* fn = nullptr;
  DISPATCH_DK(d->dim, d->k, fn = (void*)dev::small_vcycle<D_, K_, T>);
  CK(cudaLaunchCooperativeKernel(fn, dim3(d->slk_grid), dim3(dev::SLK_THREADS), args, 0, s));
  d->launches++;
}

// The V-cycle on the MG-layout buffers D (defects, copy_to_mg done), X (out).
template <typename T>
static void vcycle_levels(DeviceHierarchy* d, cudaStream_t s) {
  const int L = d->L, l0 = d->slk_ls + 1;
  T *D = MG<T>::D(d), *X = MG<T>::X(d), *Tb = MG<T>::T(d), *DV = MG<T>::DV(d);
  for (int l = L; l >= l0; --l) {
    DevLevel& v = d->lv[l];
    T *g = D + v.off, *x = X + v.off, *t = Tb + v.off, *dv = DV + v.off;
    T* gc = D + d->lv[l - 1].off;
    smooth(d, l, g, x, t, dv, true, s);                                     // 1: pre-smooth from 0
    if (res_fusable(d, l)) {                                                // 2 + 3 in one pass over the level
      res_restrict(d, l, x, g, gc, s);
    } else {
      apply_full(d, l, x, t, s);                                            // 2: t = K x
      k_restrict<dev::RES_VCYCLE>(d, l, nullptr, v.n_fam, g, t, gc, s);     // 3: d_{l-1} += P^T (d - t)
    }
    export_add(d, l - 1, gc, s);
  }
  if (d->slk_ls > 0) run_small_levels<T>(d, s);                                 // V(l_s), coarse solve included
  else coarse(d, D + d->lv[0].off, X + d->lv[0].off, Tb + d->lv[0].off, DV + d->lv[0].off, s);   // 4: coarse solve
  for (int l = l0; l <= L; ++l) {
    DevLevel& v = d->lv[l];
    T *g = D + v.off, *x = X + v.off, *t = Tb + v.off, *dv = DV + v.off;
    T* xc = X + d->lv[l - 1].off;
    import_ghosts(d, l - 1, xc, s);
    if (prolong_fusable(d, l)) {
      smooth(d, l, g, x, t, dv, false, s, (const T*)xc);                    // 5 + 6 in one pass over the level
    } else {
      k_prolongate<dev::XFER_ADD>(d, l, nullptr, v.n_fam, xc, x, s);       // 5: x += P x_{l-1}
      smooth(d, l, g, x, t, dv, false, s);                                  // 6: post-smooth
    }
  }
}

// the per-level parameters of small_vcycle (Chebyshev coefficients change with
// gmg_set_eigen): uploaded before every capture and eager cycle
static void upload_slk(DeviceHierarchy* d, cudaStream_t s) {
  if (d->slk_ls == 0) return;
  std::vector<dev::SlkLevel> h(d->slk_ls + 1);
  for (int l = 0; l <= d->slk_ls; ++l) {
    DevLevel& v = d->lv[l];
    dev::SlkLevel& q = h[l];
    std::memset(&q, 0, sizeof q);
    q.xfer = v.xfer;
    q.cls = v.cls;
    q.Dinv = d->mixed ? (const void*)v.Dinv32 : (const void*)v.Dinv;
    q.n_fam = v.n_fam;
    q.n_r1 = v.n_r1;
    q.n_pad = v.n_pad;
    q.n_owned = v.n_owned;
    q.off = v.off;
    q.off_c = l > 0 ? d->lv[l - 1].off : 0;
    q.scale = v.scale;
    const int np = d->dim == 3 ? (2 * d->k + 1) * (2 * d->k + 1) * (2 * d->k + 1) : (2 * d->k + 1) * (2 * d->k + 1);
    q.row = np + nn_of(d);
    q.m = (int)v.c1.size();
    q.fuse_pro = l > 0 && prolong_fusable(d, l) ? 1 : 0;
    for (int j = 0; j < q.m && j < 16; ++j) {
      q.c1[j] = v.c1[j];
      q.c2[j] = v.c2[j];
    }
  }
  CK(cudaMemcpyAsync(d->slk_dev, h.data(), h.size() * sizeof(dev::SlkLevel), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
}

// x1_done: the caller has formed the finest level's x_1 (fuse_x1)
static void run_vcycle_mg(DeviceHierarchy* d, cudaStream_t s, bool x1_done = false) {
  d->skip_x1 = x1_done;
  if (!d->use_graph) {
    upload_slk(d, s);
    if (d->mixed) vcycle_levels<float>(d, s);
    else vcycle_levels<double>(d, s);
    d->skip_x1 = false;
    return;
  }
  cudaGraphExec_t& ge = x1_done ? d->vgraph_x1 : d->vgraph;
  if (!ge) {
    upload_slk(d, s);
    long long before = d->launches;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(d->cap, cudaStreamCaptureModeThreadLocal));
    if (d->mixed) vcycle_levels<float>(d, d->cap);
    else vcycle_levels<double>(d, d->cap);
    CK(cudaStreamEndCapture(d->cap, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphDestroy(g));
    (x1_done ? d->per_vcycle_x1 : d->per_vcycle) = d->launches - before;
    d->launches = before;
  }
  d->skip_x1 = false;
  CK(cudaGraphLaunch(ge, s));
  d->launches += x1_done ? d->per_vcycle_x1 : d->per_vcycle;
}

// The finest level's first pre-smoothing pass x_1 = c2_0 D^-1 g can ride on
// copy_to_mg (gmg_vcycle only; GMG_FUSE_X1=0 restores the pass): that level's
// defect is complete once gathered (no restriction adds into it), the pass is a
// pure row-wise map of it, and the smoother takes the separate-pass branch there.
static bool fuse_x1(const DeviceHierarchy* d) {
  static const bool on = [] {
    const char* e = std::getenv("GMG_FUSE_X1");
    return !(e && e[0] == '0');
  }();
  const DevLevel& v = d->lv[d->L];
  return on && d->L >= 1 && d->L > d->slk_ls && v.c1.size() > 1 && v.n_pad > 0 && !(z1_enabled() && v.n_r1 > 0);
}

// leaf operator in MG layout: q = lam * Y, Y = A_leaf p (hanging nodes via E rows)
static void leaf_apply_mg(DeviceHierarchy* d, const double* p, double* q, double* partial, cudaStream_t s) {
  const int L = d->L;
  long long before = d->launches;
  CK(cudaMemcpyAsync(d->W, p, d->N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  for (int l = 1; l <= L; ++l) {
    import_ghosts(d, l - 1, d->W + d->lv[l - 1].off, s);
    k_prolongate<dev::XFER_SET_E>(d, l, d->lv[l].edge_fams, d->lv[l].n_edge, d->W + d->lv[l - 1].off,
                                  d->W + d->lv[l].off, s);
  }
  import_ghosts(d, L, d->W + d->lv[L].off, s);
  CK(cudaMemsetAsync(d->Y, 0, d->N * sizeof(double), s));
  for (int l = 0; l <= L; ++l) {
    // a level whose cells are all leaves (c3's finest) runs the family-patch
    // operator over the whole level instead of the thread-per-cell list kernel
    const DevLevel& v = d->lv[l];
    const bool all = l > 0 && v.n_fam > 0 && v.n_leaf == v.n_cells;
    k_apply(d, l, all ? nullptr : v.leaf_cells, all ? v.n_cells : v.n_leaf, d->W + v.off, d->Y + v.off, s);
  }
  for (int l = L; l >= 1; --l) {
    export_add(d, l, d->Y + d->lv[l].off, s);
    k_restrict<dev::RES_EONLY, double>(d, l, d->lv[l].edge_fams, d->lv[l].n_edge, d->Y + d->lv[l].off, nullptr,
                               d->Y + d->lv[l - 1].off, s);
  }
  export_add(d, 0, d->Y + d->lv[0].off, s);
  dev::mask_dot<<<d->nred, dev::RED_NT, 0, s>>>(d->N, d->lam_mg, d->Y, p, q, partial);
  d->launches++;
  d->per_leaf_apply = d->launches - before;
}

static double host_dot(DeviceHierarchy* d, i64 n, const double* a, const double* b, cudaStream_t s) {
  if (n > 0) {
    dev::dot_partial<<<d->nred, dev::RED_NT, 0, s>>>(n, a, b, d->partial);
    dev::reduce_final<<<1, dev::RED_NT, 0, s>>>(d->nred, d->partial, d->scal + 7);
    d->launches += 2;
  } else {
    CK(cudaMemsetAsync(d->scal + 7, 0, sizeof(double), s));
  }
  allreduce(d, d->scal + 7, 1, s);
  CK(cudaMemcpyAsync(d->hscal + 7, d->scal + 7, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return d->hscal[7];
}

// first-kind Chebyshev coefficients over [lo, hi], degree m (SURVEY c.1 step 9)
static void set_cheb_range(DevLevel& v, double lo, double hi, int m) {
  v.c1.assign(m, 0.0);
  v.c2.assign(m, 0.0);
  if (!(hi > 0)) return;
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo);
  v.c2[0] = 1.0 / theta;
  if (!(delta > 1e-14 * theta)) {        // one eigenvalue: the first step is exact
    v.c1.resize(1);
    v.c2.resize(1);
    return;
  }
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  for (int j = 1; j < m; ++j) {
    double rn = 1.0 / (2.0 * sigma - rho);
    v.c1[j] = rn * rho;
    v.c2[j] = 2.0 * rn / delta;
    rho = rn;
  }
}

static void set_cheb(DeviceHierarchy* d, int l) {
  DevLevel& v = d->lv[l];
  set_cheb_range(v, d->lo * v.lam, d->hi * v.lam, d->m);
}

// largest eigenvalue of a symmetric tridiagonal matrix (cyclic Jacobi on the
// dense matrix, m <= ~20)
static double tridiag_max_eig(const std::vector<double>& a, const std::vector<double>& b) {
  const int m = (int)a.size();
  std::vector<double> A((size_t)m * m, 0.0);
  for (int i = 0; i < m; ++i) A[(size_t)i * m + i] = a[i];
  for (int i = 1; i < m; ++i) A[(size_t)i * m + i - 1] = A[(size_t)(i - 1) * m + i] = b[i - 1];
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int i = 0; i < m; ++i)
      for (int j = i + 1; j < m; ++j) off += A[(size_t)i * m + j] * A[(size_t)i * m + j];
    if (off < 1e-300) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        double apq = A[(size_t)p * m + q];
        if (apq == 0.0) continue;
        double app = A[(size_t)p * m + p], aqq = A[(size_t)q * m + q];
        double th = (aqq - app) / (2.0 * apq);
        double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < m; ++r) {
          double arp = A[(size_t)r * m + p], arq = A[(size_t)r * m + q];
          A[(size_t)r * m + p] = c * arp - s * arq;
          A[(size_t)r * m + q] = s * arp + c * arq;
        }
        for (int r = 0; r < m; ++r) {
          double apr = A[(size_t)p * m + r], aqr = A[(size_t)q * m + r];
          A[(size_t)p * m + r] = c * apr - s * aqr;
          A[(size_t)q * m + r] = s * apr + c * aqr;
        }
      }
  }
  double mx = -1e300;
  for (int i = 0; i < m; ++i) mx = std::max(mx, A[(size_t)i * m + i]);
  return mx;
}
static double tridiag_min_eig(std::vector<double> a, std::vector<double> b) {
  for (auto& v : a) v = -v;
  for (auto& v : b) v = -v;
  return -tridiag_max_eig(a, b);
}

// CG (Jacobi preconditioned) on A^S x = v, v = (-5.5, ..., 5.5, -5.5, ...)
// over the S DoFs in canonical order, at most maxit iterations, stopping when the
// unpreconditioned residual falls below tol ||r_0||; Lanczos tridiagonal from the
// CG coefficients; its extreme eigenvalues.  Collective over ranks (global dots,
// same control flow everywhere).
static void lanczos_range(DeviceHierarchy* d, int l, int maxit, double tol, double* lo, double* hi,
                          cudaStream_t s) {
  DevLevel& v = d->lv[l];
  const i64 n = v.n;
  *lo = *hi = 0.0;
  if (v.nS_global == 0) return;
  double *r = d->X + v.off, *z = d->DV + v.off, *p = d->W + v.off, *q = d->Y + v.off;
  const int gr = (int)((n + 255) / 256);
  if (n > 0) {
    CK(cudaMemcpyAsync(r, v.eig_v.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    dev::eig_z<<<gr, 256, 0, s>>>(n, v.Dinv, r, z);
    CK(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    d->launches++;
  }
  double rz = host_dot(d, n, r, z, s);
  double r0 = std::sqrt(host_dot(d, n, r, r, s));
  std::vector<double> alphas, betas;
  if (rz == 0.0 || r0 == 0.0) return;
  for (int it = 0; it < maxit; ++it) {
    if (n > 0) CK(cudaMemsetAsync(q, 0, n * sizeof(double), s));
    apply_full(d, l, p, q, s);
    double pq = host_dot(d, n, p, q, s);
    double alpha = rz / pq;
    alphas.push_back(alpha);
    if (n > 0) {
      dev::eig_update_r<<<gr, 256, 0, s>>>(n, alpha, v.cls, q, r);
      d->launches++;
    }
    if (it == maxit - 1) break;
    if (n > 0) {
      dev::eig_z<<<gr, 256, 0, s>>>(n, v.Dinv, r, z);
      d->launches++;
    }
    double rz_new = host_dot(d, n, r, z, s);
    double rn = std::sqrt(host_dot(d, n, r, r, s));
    if (rn <= tol * r0 || rz_new == 0.0) break;
    double beta = rz_new / rz;
    betas.push_back(beta);
    if (n > 0) {
      dev::axpby<<<gr, 256, 0, s>>>(n, 1.0, z, beta, p);
      d->launches++;
    }
    rz = rz_new;
  }
  const int m = (int)alphas.size();
  std::vector<double> a(m), b(m > 0 ? m - 1 : 0);
  for (int j = 0; j < m; ++j) {
    a[j] = 1.0 / alphas[j] + (j > 0 ? betas[j - 1] / alphas[j - 1] : 0.0);
    if (j > 0) b[j - 1] = std::sqrt(betas[j - 1]) / alphas[j - 1];
  }
  *hi = tridiag_max_eig(a, b);
  *lo = tridiag_min_eig(a, b);
}

// lambda_bar of level l >= 1: min(eig_iters, n_S) iterations (reading R11)
static double eigen_estimate(DeviceHierarchy* d, int l, cudaStream_t s) {
  double lo, hi;
  lanczos_range(d, l, (int)std::min<i64>(d->eig_iters, d->lv[l].nS_global), 1e-10, &lo, &hi, s);
  return hi;
}

// P:890-895 coarse solver: Chebyshev over the full eigenvalue range of D^-1 A_0^S
// (Lanczos of a CG run to relative unpreconditioned residual 1e-3) with the smallest
// degree whose a priori bound 2 rho^m / (1 + rho^2m) is <= 1e-3 (reading R28).
static int chebyshev_degree(double kappa, double eps) {
  if (!(kappa > 1.0 + 1e-12)) return 1;
  const double rho = (std::sqrt(kappa) - 1.0) / (std::sqrt(kappa) + 1.0);
  int m = 1;
  while (2.0 * std::pow(rho, m) / (1.0 + std::pow(rho, 2 * m)) > eps && m < 100000) ++m;
  return m;
}

// ---------------------------------------------------------------- creation
DeviceHierarchy* device_create(LocalTopo& Tp, const gmg_params& prm, std::unique_ptr<Comm> comm,
                               i64 n0_global) {
  auto* d = new DeviceHierarchy();
  try {
    const bool gfam = [] {
      const char* e = std::getenv("GMG_GFAM");
      return !(e && e[0] == '0');
    }();
    // small levels in one persistent kernel (small_vcycle): levels 1..ls, see DeviceHierarchy
    int ls = 0;
    {
      // off by default: measured slower than the graph-launched per-step kernels
      // (grid barriers cost more than kernel boundaries inside a CUDA graph)
      const char* e = std::getenv("GMG_SLK");
      const bool on = e && e[0] == '1';
      i64 fam_max = 2048;
      if (const char* f = std::getenv("GMG_SLK_FAM")) fam_max = std::atoll(f);
      bool tensor_ok = true;
      if (const char* a = std::getenv("GMG_APPLY")) tensor_ok = std::string(a) != "cell";
      if (on && !comm && prm.coarse_solver == GMG_COARSE_CHOLESKY && tensor_ok && Tp.lv[0].cell_elem.empty())
        for (int l = 1; l <= Tp.L; ++l) {
          const LocalLevel& t = Tp.lv[l];
          if (!(t.n_fam > 0 && t.n_fam <= fam_max && t.cell_elem.empty() && t.cell_coef.empty() && t.fam_coef.empty()))
            break;
          ls = l;
        }
      if (ls >= Tp.L) ls = Tp.L - 1;   // the finest level stays outside (the copies to/from the MG layout)
      if (ls < 1) ls = 0;
    }
    eig_start_from_keys(Tp);                                        // rank-local builds: R10b from the keys
    const DevicePlan plan = plan_device_order(Tp, gfam, ls + 1);   // device order of the level vectors (rewrites Tp)
    if (prm.device >= 0) CK(cudaSetDevice(prm.device));
    int dev_id = 0;
    CK(cudaGetDevice(&dev_id));
    CK(cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, dev_id));
    d->comm = std::move(comm);
    GMG_REQUIRE((prm.dev_alloc == nullptr) == (prm.dev_free == nullptr), GMG_E_INVALID_ARG,
                "dev_alloc and dev_free must be given together");
    d->dev_alloc = prm.dev_alloc;
    d->dev_free = prm.dev_free;
    d->alloc_ctx = prm.alloc_ctx;
    d->dim = Tp.dim;
    d->k = Tp.k;
    d->L = Tp.L;
    d->m = prm.cheb_degree;
    d->lo = prm.cheb_lo;
    d->hi = prm.cheb_hi;
    d->eig_iters = prm.eig_iters;
    d->n0_global = n0_global;
    d->use_graph = !(prm.flags & GMG_NO_GRAPH) && (!d->comm || d->comm->capturable());
    d->mixed = (prm.flags & GMG_MIXED_PRECISION) != 0;
    d->coarse_cheb = prm.coarse_solver == GMG_COARSE_CHEBYSHEV;
    if (const char* e = std::getenv("GMG_APPLY")) d->tensor_apply = std::string(e) != "cell";
    if (const char* e = std::getenv("GMG_GF_SLOTS")) d->gf_slots = std::max(1, std::min(3, std::atoi(e)));
    GMG_REQUIRE(d->m >= 1 && d->m <= 16, GMG_E_INVALID_ARG, "cheb_degree must be in [1,16]");
    CK(cudaStreamCreateWithFlags(&d->cap, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&d->cstream, cudaStreamNonBlocking));
    if (const char* e = std::getenv("GMG_OVERLAP")) d->overlap = !(e[0] == '0');
    const int nn = Tp.dim == 2 ? (Tp.k + 1) * (Tp.k + 1) : (Tp.k + 1) * (Tp.k + 1) * (Tp.k + 1);
    d->lv.resize(Tp.L + 1);
    i64 off = 0, xmax = 1;
    for (int l = 0; l <= Tp.L; ++l) {
      const LocalLevel& t = Tp.lv[l];
      DevLevel& v = d->lv[l];
      v.n = t.n_local();
      v.n_owned = t.n_owned;
      v.n_pad = (v.n + dev::VEC_PAD - 1) / dev::VEC_PAD * dev::VEC_PAD;   // zero padding
      v.n_cells = t.n_cells;
      v.n_fam = t.n_fam;
      v.n_leaf = (i64)t.leaf_cells.size();
      v.n_edge = (i64)t.edge_fams.size();
      v.nS_global = t.nS_global;
      v.eig_v = t.eig_v;
      v.off = off;
      off += v.n_pad;
      v.ldc = (long)t.n_cells;
      std::vector<int> soa((size_t)t.n_cells * nn);
      for (i64 c = 0; c < t.n_cells; ++c)
        for (int b = 0; b < nn; ++b) soa[(size_t)b * t.n_cells + c] = t.cell_dofs[(size_t)c * nn + b];
      v.cell_dofs = d->upload(soa);
      std::vector<unsigned char> cls(v.n);
      for (i64 i = 0; i < v.n; ++i) cls[i] = t.cls[i] == CLS_E ? 1 : 0;
      v.cls = d->upload(cls);
      v.xfer = d->upload(t.xfer);
      if (!d->tensor_apply || (!t.cell_coef.empty() && t.fam_coef.empty())) {
        // cell-form family apply (config-4 level 2, or GMG_APPLY=cell): patch table
        // AoS (host) -> SoA [(2k+1)^d][n_fam] (device)
        const size_t np = Tp.dim == 3 ? (2 * Tp.k + 1) * (2 * Tp.k + 1) * (2 * Tp.k + 1) : (2 * Tp.k + 1) * (2 * Tp.k + 1);
        const size_t xr = np + nn;
        std::vector<int> fs(np * t.n_fam);
        for (size_t f = 0; f < (size_t)t.n_fam; ++f)
          for (size_t a = 0; a < np; ++a) fs[a * t.n_fam + f] = t.xfer[f * xr + a];
        v.fam_dofs = d->upload(fs);
      }
      v.leaf_cells = d->upload(t.leaf_cells);
      v.n_r1 = plan.n_r1[l];
      v.perm = d->upload(plan.perm[l]);
      v.n_fam_int = (i64)plan.fam_int[l].size();
      v.n_fam_bnd = (i64)plan.fam_bnd[l].size();
      v.n_gf_int = (i64)plan.gf_int[l].size();
      v.n_gf_bnd = (i64)plan.gf_bnd[l].size();
      v.split = v.n_fam_int + v.n_gf_int > 0;
      if (v.split) {
        v.fam_int = d->upload(plan.fam_int[l]);
        v.fam_bnd = d->upload(plan.fam_bnd[l]);
        v.gf_int = d->upload(plan.gf_int[l]);
        v.gf_bnd = d->upload(plan.gf_bnd[l]);
        CK(cudaEventCreateWithFlags(&v.ev_pack, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&v.ev_ghost, cudaEventDisableTiming));
      }
      v.n_gf = plan.n_gf[l];
      if (v.n_gf > 0) {
        v.gx = d->upload(plan.gx[l]);
        v.gr1 = d->upload(plan.gr1[l]);
        v.n_single = (i64)plan.singles[l].size();
        v.singles = d->upload(plan.singles[l]);
        if (!plan.gcoef[l].empty()) v.gcoef = d->upload(plan.gcoef[l]);
      }
      if (!t.cell_coef.empty()) v.coef = d->upload(t.cell_coef);
      if (!t.fam_coef.empty()) v.fcoef = d->upload(t.fam_coef);
      if (!t.cell_elem.empty()) v.elem = d->upload(t.cell_elem);
      v.edge_fams = d->upload(t.edge_fams);
      v.h = std::ldexp(1.0, -l);
      v.scale = Tp.dim == 3 ? v.h : 1.0;
      v.Dinv = d->alloc<double>(v.n_pad);
      CK(cudaMemset(v.Dinv, 0, v.n_pad * sizeof(double)));
      v.peers = t.peers;
      v.send_off = t.send_off;
      v.recv_off = t.recv_off;
      v.n_send = (i64)t.send_idx.size();
      v.n_recv = (i64)t.recv_idx.size();
      v.send_idx = d->upload(t.send_idx);
      v.recv_idx = d->upload(t.recv_idx);
      xmax = std::max(xmax, std::max(v.n_send, v.n_recv));
    }
    d->N = off;
    const i64 N = d->N;
    d->slk_ls = ls;
    if (ls > 0) {
      d->slk_dev = d->alloc<dev::SlkLevel>(ls + 1);
      int per_sm = 0;
      void* fn = nullptr;
      const bool f32 = (prm.flags & GMG_MIXED_PRECISION) != 0;
      if (f32) {
        DISPATCH_DK(d->dim, d->k, fn = (void*)dev::small_vcycle<D_, K_, float>);
      } else {
        DISPATCH_DK(d->dim, d->k, fn = (void*)dev::small_vcycle<D_, K_, double>);
      }
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, dev::SLK_THREADS, 0));
      int bps = 2;
      if (const char* e = std::getenv("GMG_SLK_BPS")) bps = std::max(1, std::atoi(e));
      d->slk_grid = std::max(1, std::min(per_sm, bps)) * d->sms;
      if (const char* e = std::getenv("GMG_SLK_GRID"))   // a fixed number of CTAs (few CTAs: cheaper barriers)
        d->slk_grid = std::max(1, std::min(std::atoi(e), per_sm * d->sms));
      if (per_sm < 1) d->slk_ls = 0;
    }
    for (double** p : {&d->D, &d->X, &d->T, &d->DV, &d->W, &d->Y, &d->cx, &d->cr, &d->cp, &d->cq, &d->cz}) {
      *p = d->alloc<double>(N);
      CK(cudaMemset(*p, 0, N * sizeof(double)));
    }
    d->sbuf = d->alloc<double>(xmax);
    d->rbuf = d->alloc<double>(xmax);
    // lambda mask and leaf <-> MG maps (owned leaf DoFs of this rank)
    std::vector<unsigned char> lam(N, 0);
    GMG_REQUIRE(N < ((i64)1 << 31), GMG_E_INVALID_ARG, "MG layout exceeds 2^31 entries on one rank");
    std::vector<int> m2l(N, -1), l2m(Tp.n_leaf_owned);
    for (int l = 0; l <= Tp.L; ++l)
      for (i64 i = 0; i < Tp.lv[l].n_local(); ++i) lam[d->lv[l].off + i] = Tp.lv[l].lam[i];
    for (i64 g = 0; g < Tp.n_leaf_owned; ++g) {
      i64 m = d->lv[Tp.leaf_level[g]].off + Tp.leaf_local[g];
      l2m[g] = (int)m;
      m2l[m] = (int)g;
    }
    d->n_leaf = Tp.n_leaf_owned;
    d->lam_mg = d->upload(lam);
    d->mg_to_leaf = d->upload(m2l);
    d->leaf_to_mg = d->upload(l2m);
    d->nred = d->sms * 4;
    d->partial = d->alloc<double>(d->nred);
    d->scal = d->alloc<double>(16);
    CK(cudaMemset(d->scal, 0, 16 * sizeof(double)));
    CK(cudaMallocHost(&d->hscal, 16 * sizeof(double)));
    cudaStream_t s = d->cap;
    // diagonal and D^-1 on owned S rows (ghost contributions added to owners)
    int* bad = d->alloc<int>(1);
    CK(cudaMemset(bad, 0, sizeof(int)));
    for (int l = 0; l <= Tp.L; ++l) {
      DevLevel& v = d->lv[l];
      if (v.n_cells > 0 && v.elem) {
        const int nn = d->dim == 3 ? (d->k + 1) * (d->k + 1) * (d->k + 1) : (d->k + 1) * (d->k + 1);
        DISPATCH_DK(d->dim, d->k,
                    (dev::cell_diag_dense<D_, K_><<<(int)((v.n_cells * nn + 127) / 128), 128, 0, s>>>(
                        (int)v.n_cells, v.cell_dofs, v.ldc, v.elem, v.Dinv)));
        d->launches++;
      } else if (v.n_cells > 0) {
        int grid = (int)((v.n_cells + 127) / 128);
        DISPATCH_DK(d->dim, d->k,
                    (dev::cell_diag<D_, K_><<<grid, 128, 0, s>>>((int)v.n_cells, v.cell_dofs, v.ldc, v.coef, v.scale,
                                                                 v.Dinv)));
        d->launches++;
      }
      export_add(d, l, v.Dinv, s);
      if (v.n_owned > 0) {
        dev::invert_diag<<<(int)((v.n_owned + 255) / 256), 256, 0, s>>>(v.n_owned, v.cls, v.Dinv, bad);
        d->launches++;
      }
    }
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    GMG_REQUIRE(hbad == 0, GMG_E_ZERO_DIAG, "zero or negative diagonal on an S row");
    // coarse matrix A_0^S (all level-0 DoFs owned by rank 0): columns by a
    // collective apply of K_0 to unit vectors; dense Cholesky on rank 0
    if (!d->coarse_cheb) {
      DevLevel& v0 = d->lv[0];
      const int n0 = (int)n0_global;
      d->nS0 = (int)v0.n_owned;
      GMG_REQUIRE(n0 <= 4096, GMG_E_INVALID_ARG, "coarse level too large for the dense solver");
      std::vector<double> A((size_t)n0 * n0), e(std::max<i64>(v0.n, 1));
      double *xe = d->X + v0.off, *ye = d->Y + v0.off;
      for (int j = 0; j < n0; ++j) {
        std::fill(e.begin(), e.end(), 0.0);
        if (d->nS0 > 0) e[j] = 1.0;
        if (v0.n > 0) {
          CK(cudaMemcpyAsync(xe, e.data(), v0.n * sizeof(double), cudaMemcpyHostToDevice, s));
          CK(cudaMemsetAsync(ye, 0, v0.n * sizeof(double), s));
        }
        apply_full(d, 0, xe, ye, s);
        if (d->nS0 > 0)
          CK(cudaMemcpyAsync(A.data() + (size_t)j * n0, ye, n0 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
      }
      if (d->nS0 > 0) {
        std::vector<double> Lm((size_t)n0 * n0, 0.0);
        for (int i = 0; i < n0; ++i)
          for (int j = 0; j <= i; ++j) {
            double sum = 0.5 * (A[(size_t)i * n0 + j] + A[(size_t)j * n0 + i]);
            for (int q = 0; q < j; ++q) sum -= Lm[(size_t)i * n0 + q] * Lm[(size_t)j * n0 + q];
            if (i == j) {
              GMG_REQUIRE(sum > 0.0, GMG_E_SINGULAR_COARSE, "coarse matrix not SPD");
              Lm[(size_t)i * n0 + i] = std::sqrt(sum);
            } else {
              Lm[(size_t)i * n0 + j] = sum / Lm[(size_t)j * n0 + j];
            }
          }
        std::vector<double> inv((size_t)n0 * n0);
        for (int c = 0; c < n0; ++c) {
          std::vector<double> y(n0), x(n0);
          for (int i = 0; i < n0; ++i) {
            double sum = (i == c) ? 1.0 : 0.0;
            for (int q = 0; q < i; ++q) sum -= Lm[(size_t)i * n0 + q] * y[q];
            y[i] = sum / Lm[(size_t)i * n0 + i];
          }
          for (int i = n0 - 1; i >= 0; --i) {
            double sum = y[i];
            for (int q = i + 1; q < n0; ++q) sum -= Lm[(size_t)q * n0 + i] * x[q];
            x[i] = sum / Lm[(size_t)i * n0 + i];
          }
          for (int i = 0; i < n0; ++i) inv[(size_t)i * n0 + c] = x[i];
        }
        std::vector<int> idx(n0);
        for (int i = 0; i < n0; ++i) idx[i] = i;
        d->coarse_idx = d->upload(idx);
        d->coarse_inv = d->upload(inv);
      }
    }
    // eigenvalue estimates (levels >= 1), collective
    for (int l = 1; l <= Tp.L; ++l) {
      d->lv[l].lam = eigen_estimate(d, l, s);
      set_cheb(d, l);
    }
    // prolongation fusion per level, collectively: every rank has R1 rows there
    {
      const int nl = Tp.L + 1;
      GMG_REQUIRE(nl <= 64 && nl <= d->nred, GMG_E_INVALID_ARG, "too many levels");
      std::vector<double> miss(nl);
      for (int l = 0; l < nl; ++l) miss[l] = d->lv[l].n_r1 > 0 ? 0.0 : 1.0;
      CK(cudaMemcpyAsync(d->partial, miss.data(), nl * sizeof(double), cudaMemcpyHostToDevice, s));
      allreduce(d, d->partial, nl, s);
      CK(cudaMemcpyAsync(miss.data(), d->partial, nl * sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int l = 0; l < nl; ++l) d->lv[l].fuse_pro = l > 0 && miss[l] == 0.0;
      // residual + restriction fusion (TA_RES) per level, collectively: it drops the
      // level's export-add of t, so either every rank runs it or none
      for (int l = 0; l < nl; ++l) {
        const DevLevel& v = d->lv[l];
        miss[l] = l > 0 && d->tensor_apply && !v.elem && (v.coef == nullptr || v.fcoef != nullptr) ? 0.0 : 1.0;
      }
      CK(cudaMemcpyAsync(d->partial, miss.data(), nl * sizeof(double), cudaMemcpyHostToDevice, s));
      allreduce(d, d->partial, nl, s);
      CK(cudaMemcpyAsync(miss.data(), d->partial, nl * sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int l = 0; l < nl; ++l) d->lv[l].fuse_res = miss[l] == 0.0;
    }
    if (d->coarse_cheb) {
      DevLevel& v0 = d->lv[0];
      lanczos_range(d, 0, (int)std::max<i64>(v0.nS_global, 1), 1e-3, &d->coarse_lo, &d->coarse_hi, s);
      const int m0 = d->coarse_hi > 0 ? chebyshev_degree(d->coarse_hi / d->coarse_lo, 1e-3) : 0;
      set_cheb_range(v0, d->coarse_lo, d->coarse_hi, m0);
    }
    // restore the work buffers to zero (T must be zero between applies)
    for (double* p : {d->X, d->T, d->DV, d->W, d->Y}) CK(cudaMemsetAsync(p, 0, N * sizeof(double), s));
    if (d->mixed) {   // fp32 V-cycle buffers; D^-1 rounded once from the fp64 diagonal
      for (float** p : {&d->D32, &d->X32, &d->T32, &d->DV32}) {
        *p = d->alloc<float>(N);
        CK(cudaMemsetAsync(*p, 0, N * sizeof(float), s));
      }
      for (int l = 0; l <= Tp.L; ++l) {
        DevLevel& v = d->lv[l];
        v.Dinv32 = d->alloc<float>(v.n_pad);
        dev::cast_vec<float><<<d->vgrid(v.n_pad), 256, 0, s>>>(v.n_pad, v.Dinv, v.Dinv32);
        d->launches++;
      }
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
  } catch (...) {
    device_destroy(d);
    throw;
  }
  return d;
}

long long device_mg_len(const DeviceHierarchy* d) { return d ? (long long)d->N : 0; }
long long device_small_levels(const DeviceHierarchy* d) { return d ? (long long)d->slk_ls : 0; }

void comm_allreduce_host(Comm* comm, std::vector<double>& v) {
  if (!comm || v.empty()) return;
  double* buf = nullptr;
  cudaStream_t s = nullptr;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  try {
    CK(cudaMalloc(&buf, v.size() * sizeof(double)));
    CK(cudaMemcpyAsync(buf, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    comm->allreduce(buf, (int)v.size(), s);
    CK(cudaMemcpyAsync(v.data(), buf, v.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  } catch (...) {
    if (buf) cudaFree(buf);
    cudaStreamDestroy(s);
    throw;
  }
  cudaFree(buf);
  cudaStreamDestroy(s);
}

long long device_level_gf(const DeviceHierarchy* d, int level) {
  return d && level >= 0 && level < (int)d->lv.size() ? (long long)d->lv[level].n_gf : 0;
}

long long device_level_r1(const DeviceHierarchy* d, int level) {
  return d && level >= 0 && level < (int)d->lv.size() ? (long long)d->lv[level].n_r1 : 0;
}

void device_destroy(DeviceHierarchy* d) {
  if (!d) return;
  cudaDeviceSynchronize();
  if (d->vgraph) cudaGraphExecDestroy(d->vgraph);
  if (d->vgraph_x1) cudaGraphExecDestroy(d->vgraph_x1);
  for (cudaEvent_t e : d->evpool) cudaEventDestroy(e);
  for (auto& v : d->lv) {
    if (v.ev_pack) cudaEventDestroy(v.ev_pack);
    if (v.ev_ghost) cudaEventDestroy(v.ev_ghost);
  }
  if (d->cstream) cudaStreamDestroy(d->cstream);
  for (auto& a : d->allocs) {
    if (d->dev_free) d->dev_free(a.first, a.second, nullptr, d->alloc_ctx);
    else cudaFree(a.first);
  }
  if (d->hscal) cudaFreeHost(d->hscal);
  if (d->cap) cudaStreamDestroy(d->cap);
  delete d;
}

// ---------------------------------------------------------------- API ops
void device_vcycle(DeviceHierarchy* d, const double* b, double* x, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const bool fx1 = fuse_x1(d);
  {
  const size_t vb = d->mixed ? 4 : 8;
  Prof pr(d, s, GMG_K_COPY_MG, -1, 8.0 * (double)d->n_leaf + (4.0 + vb) * (double)d->N +
                                      (fx1 ? 2.0 * vb * (double)d->lv[d->L].n_pad : 0.0));
  const DevLevel& vL = d->lv[d->L];
  const i64 lo = fx1 ? vL.off : 0, hi = fx1 ? vL.off + vL.n_pad : 0;
  const double c20 = fx1 ? vL.c2[0] : 0.0;
  if (d->mixed)                                                                                 // copy_to_mg
    dev::gather_to_mg<float><<<grid4(d->N), 256, 0, s>>>(d->N, d->mg_to_leaf, b, d->D32, lo, hi, vL.Dinv32, d->X32, c20);
  else
    dev::gather_to_mg<double><<<grid4(d->N), 256, 0, s>>>(d->N, d->mg_to_leaf, b, d->D, lo, hi, vL.Dinv, d->X, c20);
  d->launches++;
  }
  run_vcycle_mg(d, s, fx1);
  if (d->n_leaf) {                                                                              // copy_from_mg
    Prof pr(d, s, GMG_K_COPY_MG, -1, (4.0 + 8.0 + (d->mixed ? 4 : 8)) * (double)d->n_leaf);
    if (d->mixed) dev::gather_from_mg<float><<<grid4(d->n_leaf), 256, 0, s>>>(d->n_leaf, d->leaf_to_mg, d->X32, x);
    else dev::gather_from_mg<double><<<grid4(d->n_leaf), 256, 0, s>>>(d->n_leaf, d->leaf_to_mg, d->X, x);
    d->launches++;
  }
  CK(cudaPeekAtLastError());
}

// z = V(r) (MG layout, fp64 in and out; the V-cycle itself in fp32 if mixed), (r, z) partials
static void precondition(DeviceHierarchy* d, cudaStream_t s) {
  const i64 N = d->N;
  if (d->mixed) {
    dev::cast_vec<float><<<d->vgrid(N), 256, 0, s>>>(N, d->cr, d->D32);
    d->launches++;
  } else {
    CK(cudaMemcpyAsync(d->D, d->cr, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  run_vcycle_mg(d, s);
  if (d->mixed) dev::mask_copy_dot<float><<<d->nred, dev::RED_NT, 0, s>>>(N, d->lam_mg, d->X32, d->cr, d->cz, d->partial);
  else dev::mask_copy_dot<double><<<d->nred, dev::RED_NT, 0, s>>>(N, d->lam_mg, d->X, d->cr, d->cz, d->partial);
  d->launches++;
}

static void global_dot_into(DeviceHierarchy* d, int slot, cudaStream_t s) {
  dev::reduce_final<<<1, dev::RED_NT, 0, s>>>(d->nred, d->partial, d->scal + slot);
  d->launches++;
  allreduce(d, d->scal + slot, 1, s);
}

int device_solve_cg(DeviceHierarchy* d, const double* b, double* x, double rtol, int max_it, int* iters,
                    double* rel_res, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const i64 N = d->N;
  const int gr = d->vgrid(N);
  // r = b (MG layout), x = 0
  dev::gather_to_mg<double><<<grid4(N), 256, 0, s>>>(N, d->mg_to_leaf, b, d->cr);
  CK(cudaMemsetAsync(d->cx, 0, N * sizeof(double), s));
  d->launches++;
  double nb = std::sqrt(host_dot(d, N, d->cr, d->cr, s));
  int it = 0;
  double rel = nb > 0 ? 1.0 : 0.0;
  int status = 0;
  if (nb > 0) {
    // z = V(r); p = z; rz = (r, z) -> scal[0]
    precondition(d, s);
    global_dot_into(d, 0, s);
    CK(cudaMemcpyAsync(d->cp, d->cz, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    status = 1;
    for (it = 1; it <= max_it; ++it) {
      leaf_apply_mg(d, d->cp, d->cq, d->partial, s);                           // q = A p, (p,q)
      global_dot_into(d, 1, s);
      dev::cg_update_xr<<<d->nred, dev::RED_NT, 0, s>>>(N, d->scal, d->cp, d->cq, d->cx, d->cr, d->partial);
      d->launches++;
      global_dot_into(d, 3, s);
      CK(cudaMemcpyAsync(d->hscal + 3, d->scal + 3, sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      rel = std::sqrt(d->hscal[3]) / nb;
      if (rel <= rtol) {
        status = 0;
        break;
      }
      if (it == max_it) break;
      precondition(d, s);                                                       // z = V(r)
      global_dot_into(d, 2, s);
      dev::cg_update_p<<<gr, 256, 0, s>>>(N, d->scal, d->cz, d->cp);            // p = z + beta p
      dev::copy_scalar<<<1, 1, 0, s>>>(d->scal + 2, d->scal + 0);
      d->launches += 2;
    }
    if (it > max_it) it = max_it;
  }
  if (d->n_leaf) {
    dev::gather_from_mg<double><<<grid4(d->n_leaf), 256, 0, s>>>(d->n_leaf, d->leaf_to_mg, d->cx, x);
    d->launches++;
  }
  CK(cudaPeekAtLastError());
  if (iters) *iters = it;
  if (rel_res) *rel_res = rel;
  return status;
}

void device_rhs_constant(DeviceHierarchy* d, double f, double* b, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemsetAsync(d->Y, 0, d->N * sizeof(double), s));
  for (int l = 0; l <= d->L; ++l) {
    DevLevel& v = d->lv[l];
    if (v.n_leaf == 0) continue;
    double fh = f * std::pow(v.h, d->dim);
    int grid = (int)((v.n_leaf + 127) / 128);
    DISPATCH_DK(d->dim, d->k, (dev::cell_load<D_, K_><<<grid, 128, 0, s>>>((int)v.n_leaf, v.leaf_cells, v.cell_dofs,
                                                                            v.ldc, fh, d->Y + v.off)));
    d->launches++;
  }
  for (int l = d->L; l >= 1; --l) {
    export_add(d, l, d->Y + d->lv[l].off, s);
    k_restrict<dev::RES_EONLY, double>(d, l, d->lv[l].edge_fams, d->lv[l].n_edge, d->Y + d->lv[l].off, nullptr,
                               d->Y + d->lv[l - 1].off, s);
  }
  export_add(d, 0, d->Y + d->lv[0].off, s);
  if (d->n_leaf) {
    dev::gather_from_mg<double><<<grid4(d->n_leaf), 256, 0, s>>>(d->n_leaf, d->leaf_to_mg, d->Y, b);
    d->launches++;
  }
  CK(cudaPeekAtLastError());
}

static void need_single(const DeviceHierarchy* d) {
  GMG_REQUIRE(!d->comm, GMG_E_STATE, "single-operator entry points are defined for n_ranks == 1");
}

// The single-operator entry points take level vectors in the rank-local level
// order (= global order for one rank) and permute to the device order
// (plan.hpp) at the boundary, through the W / Y work buffers.
static void to_dev(DeviceHierarchy* d, int l, const double* src, double* dst, cudaStream_t s) {
  DevLevel& v = d->lv[l];
  CK(cudaMemsetAsync(dst, 0, v.n_pad * sizeof(double), s));
  if (v.n) {
    dev::permute_in<<<(int)((v.n + 255) / 256), 256, 0, s>>>(v.n, v.perm, src, dst);
    d->launches++;
  }
}
static void from_dev(DeviceHierarchy* d, int l, const double* src, double* dst, cudaStream_t s) {
  DevLevel& v = d->lv[l];
  if (v.n) {
    dev::permute_out<<<(int)((v.n + 255) / 256), 256, 0, s>>>(v.n, v.perm, src, dst);
    d->launches++;
  }
}

void device_level_apply(DeviceHierarchy* d, int l, const double* x, double* y, void* stream) {
  need_single(d);
  cudaStream_t s = (cudaStream_t)stream;
  DevLevel& v = d->lv[l];
  double *xp = d->W + v.off, *yp = d->Y + v.off;
  to_dev(d, l, x, xp, s);
  CK(cudaMemsetAsync(yp, 0, v.n_pad * sizeof(double), s));
  k_apply(d, l, nullptr, v.n_cells, (const double*)xp, yp, s);
  from_dev(d, l, yp, y, s);
  CK(cudaPeekAtLastError());
}

void device_level_apply_kernel(DeviceHierarchy* d, int l, const double* x, double* y, void* stream) {
  // rank-local kernel only (vectors of the local length n_owned + n_ghost in the
  // device order), no exchange
  DevLevel& v = d->lv[l];
  k_apply(d, l, nullptr, v.n_cells, x, y, (cudaStream_t)stream);
  CK(cudaPeekAtLastError());
}

void device_level_apply_kernel_f32(DeviceHierarchy* d, int l, const float* x, float* y, void* stream) {
  DevLevel& v = d->lv[l];
  k_apply(d, l, nullptr, v.n_cells, x, y, (cudaStream_t)stream);
  CK(cudaPeekAtLastError());
}

void device_restrict(DeviceHierarchy* d, int l, const double* r, double* dc, void* stream) {
  need_single(d);
  cudaStream_t s = (cudaStream_t)stream;
  double *rp = d->W + d->lv[l].off, *cp = d->Y + d->lv[l - 1].off;
  to_dev(d, l, r, rp, s);
  to_dev(d, l - 1, dc, cp, s);
  k_restrict<dev::RES_PLAIN, double>(d, l, nullptr, d->lv[l].n_fam, rp, nullptr, cp, s);
  from_dev(d, l - 1, cp, dc, s);
  CK(cudaPeekAtLastError());
}

void device_prolongate(DeviceHierarchy* d, int l, const double* xc, double* xf, void* stream) {
  need_single(d);
  cudaStream_t s = (cudaStream_t)stream;
  double *cp = d->W + d->lv[l - 1].off, *fp = d->Y + d->lv[l].off;
  to_dev(d, l - 1, xc, cp, s);
  to_dev(d, l, xf, fp, s);
  k_prolongate<dev::XFER_ADD>(d, l, nullptr, d->lv[l].n_fam, (const double*)cp, fp, s);
  from_dev(d, l, fp, xf, s);
  CK(cudaPeekAtLastError());
}

void device_leaf_apply(DeviceHierarchy* d, const double* u, double* v, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int gr = d->vgrid(d->N);
  dev::gather_to_mg<double><<<grid4(d->N), 256, 0, s>>>(d->N, d->mg_to_leaf, u, d->cp);
  d->launches++;
  leaf_apply_mg(d, d->cp, d->cq, d->partial, s);
  if (d->n_leaf) {
    dev::gather_from_mg<double><<<grid4(d->n_leaf), 256, 0, s>>>(d->n_leaf, d->leaf_to_mg, d->cq, v);
    d->launches++;
  }
  CK(cudaPeekAtLastError());
}

void device_level_smooth(DeviceHierarchy* d, int l, const double* g, double* x, int x_zero, void* stream) {
  need_single(d);
  cudaStream_t s = (cudaStream_t)stream;
  DevLevel& v = d->lv[l];
  GMG_REQUIRE(l >= 1, GMG_E_INVALID_ARG, "no smoother on level 0");
  double* gg = d->W + v.off;
  double* xx = d->Y + v.off;
  to_dev(d, l, g, gg, s);
  if (x_zero) CK(cudaMemsetAsync(xx, 0, v.n_pad * sizeof(double), s));
  else to_dev(d, l, x, xx, s);
  smooth(d, l, (const double*)gg, xx, d->T + v.off, d->DV + v.off, x_zero != 0, s);
  from_dev(d, l, xx, x, s);
  CK(cudaMemsetAsync(gg, 0, v.n_pad * sizeof(double), s));
  CK(cudaMemsetAsync(xx, 0, v.n_pad * sizeof(double), s));
  CK(cudaPeekAtLastError());
}

void device_level_diagonal(DeviceHierarchy* d, int l, double* diag, void* stream) {
  need_single(d);
  cudaStream_t s = (cudaStream_t)stream;
  DevLevel& v = d->lv[l];
  if (v.n == 0) return;
  double* yp = d->Y + v.off;
  dev::recip_s<<<(int)((v.n + 255) / 256), 256, 0, s>>>(v.n, v.cls, v.Dinv, yp);
  d->launches++;
  from_dev(d, l, yp, diag, s);
  CK(cudaPeekAtLastError());
}

double device_get_eigen(const DeviceHierarchy* d, int l) { return d->lv[l].lam; }

void device_coarse_chebyshev(const DeviceHierarchy* d, double* lo, double* hi, int* degree) {
  *lo = d->coarse_lo;
  *hi = d->coarse_hi;
  *degree = d->coarse_cheb ? (int)d->lv[0].c1.size() : 0;
}

void device_set_eigen(DeviceHierarchy* d, int l, double lam) {
  d->lv[l].lam = lam;
  set_cheb(d, l);
  if (d->vgraph) {   // coefficients are baked into the graph: re-capture
    cudaGraphExecDestroy(d->vgraph);
    d->vgraph = nullptr;
  }
  if (d->vgraph_x1) {
    cudaGraphExecDestroy(d->vgraph_x1);
    d->vgraph_x1 = nullptr;
  }
}

// gmg_profile_vcycle: n_rep eager V-cycles (no graph) with every launch bracketed
// by events; per (kind, level): launches, summed seconds, bytes per launch.
int device_profile_vcycle(DeviceHierarchy* d, const double* b, double* x, int n_rep, gmg_kernel_stat* out,
                          int max_out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<DeviceHierarchy::ProfRec> recs;
  const bool graph = d->use_graph;
  CK(cudaStreamSynchronize(s));
  d->use_graph = false;
  d->prof = &recs;
  d->evnext = 0;
  try {
    for (int r = 0; r < n_rep; ++r) device_vcycle(d, b, x, stream);
    CK(cudaStreamSynchronize(s));
  } catch (...) {
    d->prof = nullptr;
    d->use_graph = graph;
    throw;
  }
  d->prof = nullptr;
  d->use_graph = graph;
  std::vector<gmg_kernel_stat> agg;
  for (auto& r : recs) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    gmg_kernel_stat* e = nullptr;
    for (auto& q : agg)
      if (q.kind == r.kind && q.level == r.level) e = &q;
    if (!e) {
      agg.push_back(gmg_kernel_stat{r.kind, r.level, 0, 0.0, r.bytes, r.bytes_layout});
      e = &agg.back();
    }
    e->launches += 1;
    e->seconds += 1e-3 * ms;
  }
  const int n = (int)agg.size();
  for (int i = 0; i < n && i < max_out; ++i) out[i] = agg[i];
  return n;
}

long long device_launches(const DeviceHierarchy* d) { return d->launches; }
void device_launch_profile(const DeviceHierarchy* d, long long* pv, long long* pl) {
  // the graph gmg_vcycle launches (its x_1 variant when that is in use), else the CG's
  *pv = d->per_vcycle_x1 ? d->per_vcycle_x1 : d->per_vcycle;
  *pl = d->per_leaf_apply;
}

}  // namespace gmg
