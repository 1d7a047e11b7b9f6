// C ABI of libgmg (include/gmg.h): argument checks, handle management and the
// translation of internal errors into gmg_status codes.
#include <cmath>
#include <memory>
#include <new>

#include "comm.hpp"
#include "device.hpp"
#include "forest.hpp"

struct gmg_forest {
  gmg::Forest f;
};
struct gmg_partitioning {
  const gmg_forest* forest;
  gmg::Partition p;
};
// Global sizes reported by gmg_hierarchy_info: from the global Topology, or, for
// rank-local builds (GMG_RANK_LOCAL), the per-rank counts summed over the ranks.
struct GlobalSizes {
  int dim = 2, k = 2, L = 0, n_ranks = 1;
  gmg::i64 n_leaf_nodes = -1, n_leaf_free = -1, hanging = -1, dirichlet = -1, n0 = 0;
  std::vector<gmg::i64> dofs, cells, fams, S, E, B, leaf_cells;
};

struct gmg_hierarchy {
  gmg::Topology topo;          // global level numbering (empty for GMG_RANK_LOCAL builds)
  gmg::LocalTopo local;
  GlobalSizes sz;
  gmg_params prm{};
  gmg::DeviceHierarchy* dev = nullptr;
  ~gmg_hierarchy() { gmg::device_destroy(dev); }
};

namespace {
thread_local std::string g_err;

template <class F>
gmg_status guard(F&& fn) {
  try {
    fn();
    return GMG_OK;
  } catch (const gmg::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return GMG_E_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GMG_E_STATE;
  } catch (...) {
    g_err = "unknown error";
    return GMG_E_STATE;
  }
}

#define NEED(p) GMG_REQUIRE((p) != nullptr, GMG_E_INVALID_ARG, #p " is NULL")
// leaf vectors of this rank: NULL is legal when the rank owns no leaf DoF (zero-size
// vectors, e.g. more ranks than leaves); every rank still joins the collectives
#define NEED_LEAF(h, p) \
  GMG_REQUIRE((p) != nullptr || (h)->local.n_leaf_owned == 0, GMG_E_INVALID_ARG, #p " is NULL")

gmg::DeviceHierarchy* need_dev(gmg_hierarchy* h) {
  GMG_REQUIRE(h->dev != nullptr, GMG_E_STATE, "hierarchy has no device data (GMG_HOST_ONLY)");
  return h->dev;
}
void need_level(const gmg_hierarchy* h, int level) {
  GMG_REQUIRE(level >= 0 && level <= h->sz.L, GMG_E_INVALID_ARG, "level out of range");
}
void need_global(const gmg_hierarchy* h) {
  GMG_REQUIRE(!h->local.rank_local, GMG_E_STATE,
              "global level numbering not available for a GMG_RANK_LOCAL hierarchy (use gmg_export_local_level)");
}
}  // namespace

extern "C" {

const char* gmg_last_error(void) { return g_err.c_str(); }
int gmg_abi_version(void) { return 2; }

gmg_status gmg_forest_create(int dim, int n_trees, const int32_t* tree_xyz, int64_t n_leaves,
                             const int32_t* leaf_tree, const int8_t* leaf_level, const uint64_t* leaf_morton,
                             uint32_t flags, gmg_forest** out) {
  return guard([&] {
    NEED(out);
    auto f = std::make_unique<gmg_forest>();
    f->f = gmg::forest_create(dim, n_trees, tree_xyz, n_leaves, leaf_tree, leaf_level, leaf_morton, flags);
    *out = f.release();
  });
}

gmg_status gmg_forest_generate(const gmg_recipe* r, gmg_forest** out) {
  return guard([&] {
    NEED(r);
    NEED(out);
    auto f = std::make_unique<gmg_forest>();
    f->f = gmg::forest_generate(*r);
    *out = f.release();
  });
}

gmg_status gmg_forest_sequence(int dim, gmg_sequence kind, int L, gmg_forest** out) {
  return guard([&] {
    NEED(out);
    auto f = std::make_unique<gmg_forest>();
    f->f = gmg::forest_sequence(dim, kind, L);
    *out = f.release();
  });
}

gmg_status gmg_forest_destroy(gmg_forest* f) {
  delete f;
  return GMG_OK;
}

gmg_status gmg_forest_info(const gmg_forest* f, int* dim, int* n_trees, int64_t* n_leaves, int* max_level) {
  return guard([&] {
    NEED(f);
    if (dim) *dim = f->f.dim;
    if (n_trees) *n_trees = (int)f->f.trees.size();
    if (n_leaves) *n_leaves = f->f.n_leaves();
    if (max_level) *max_level = f->f.L;
  });
}

gmg_status gmg_export_leaves(const gmg_forest* fh, int32_t* leaf_tree, int8_t* leaf_level, uint64_t* leaf_morton) {
  return guard([&] {
    NEED(fh);
    const gmg::Forest& f = fh->f;
    for (gmg::i64 i = 0; i < f.n_leaves(); ++i) {
      int l = f.level[i];
      gmg::Vec3 tp{f.gc[i][0] >> l, f.gc[i][1] >> l, f.gc[i][2] >> l};
      int t = f.tree_of(tp);
      gmg::Vec3 loc{f.gc[i][0] - (tp[0] << l), f.gc[i][1] - (tp[1] << l), f.gc[i][2] - (tp[2] << l)};
      if (leaf_tree) leaf_tree[i] = t;
      if (leaf_level) leaf_level[i] = (int8_t)l;
      if (leaf_morton) leaf_morton[i] = gmg::morton(f.dim, loc);
    }
  });
}

gmg_status gmg_partition(const gmg_forest* f, int n_ranks, gmg_partitioning** out) {
  return guard([&] {
    NEED(f);
    NEED(out);
    auto p = std::make_unique<gmg_partitioning>();
    p->forest = f;
    p->p = gmg::make_partition(f->f, n_ranks);
    *out = p.release();
  });
}

gmg_status gmg_partition_mode(const gmg_forest* f, int n_ranks, int mode, gmg_partitioning** out) {
  return guard([&] {
    NEED(f);
    NEED(out);
    auto p = std::make_unique<gmg_partitioning>();
    p->forest = f;
    p->p = gmg::make_partition(f->f, n_ranks, mode);
    *out = p.release();
  });
}

gmg_status gmg_partition_ex(const gmg_forest* f, int n_ranks, int mode, int64_t coarse_cells, gmg_partitioning** out) {
  return guard([&] {
    NEED(f);
    NEED(out);
    GMG_REQUIRE(coarse_cells >= 0, GMG_E_INVALID_ARG, "coarse_cells must be >= 0");
    auto p = std::make_unique<gmg_partitioning>();
    p->forest = f;
    p->p = gmg::make_partition(f->f, n_ranks, mode, coarse_cells);
    *out = p.release();
  });
}

gmg_status gmg_partition_destroy(gmg_partitioning* p) {
  delete p;
  return GMG_OK;
}

gmg_status gmg_partition_model(const gmg_partitioning* p, int64_t W0_override, gmg_model* out) {
  return guard([&] {
    NEED(p);
    NEED(out);
    *out = gmg::partition_model(p->p, W0_override);
  });
}

gmg_status gmg_export_tallies(const gmg_partitioning* p, int64_t* N_lp) {
  return guard([&] {
    NEED(p);
    NEED(N_lp);
    const int P = p->p.n_ranks;
    for (size_t l = 0; l < p->p.levels.size(); ++l) {
      for (int r = 0; r < P; ++r) N_lp[l * P + r] = 0;
      for (auto o : p->p.levels[l].owner) N_lp[l * P + o]++;
    }
  });
}

gmg_status gmg_export_level_cells(const gmg_partitioning* p, int level, int64_t* n, uint64_t* key, int32_t* owner,
                                  uint8_t* is_leaf) {
  return guard([&] {
    NEED(p);
    NEED(n);
    GMG_REQUIRE(level >= 0 && level < (int)p->p.levels.size(), GMG_E_INVALID_ARG, "level out of range");
    const auto& lc = p->p.levels[level];
    *n = (int64_t)lc.key.size();
    for (size_t c = 0; c < lc.key.size(); ++c) {
      if (key) key[c] = lc.key[c];
      if (owner) owner[c] = lc.owner[c];
      if (is_leaf) is_leaf[c] = lc.leaf[c];
    }
  });
}

void gmg_params_default(gmg_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof *p);
  p->k = 2;
  p->cheb_degree = 4;
  p->cheb_lo = 0.08;
  p->cheb_hi = 1.2;
  p->eig_iters = 10;
  p->coef_level2 = nullptr;
  p->rank = 0;
  p->n_ranks = 1;
  p->nccl_comm = nullptr;
  p->device = -1;
  p->flags = 0;
  p->coarse_solver = GMG_COARSE_CHOLESKY;
  p->dev_alloc = nullptr;
  p->dev_free = nullptr;
  p->alloc_ctx = nullptr;
}

gmg_status gmg_setup(const gmg_forest* f, const gmg_partitioning* p, const gmg_params* prm, gmg_hierarchy** out) {
  return guard([&] {
    NEED(f);
    NEED(p);
    NEED(prm);
    NEED(out);
    GMG_REQUIRE(p->forest == f, GMG_E_INVALID_ARG, "partition was not built from this forest");
    GMG_REQUIRE(prm->n_ranks == p->p.n_ranks, GMG_E_INVALID_ARG, "params.n_ranks != partition n_ranks");
    GMG_REQUIRE(prm->rank >= 0 && prm->rank < prm->n_ranks, GMG_E_INVALID_ARG, "rank out of range");
    GMG_REQUIRE(prm->cheb_degree >= 1 && prm->cheb_degree <= 16, GMG_E_INVALID_ARG, "cheb_degree");
    GMG_REQUIRE(prm->cheb_lo > 0 && prm->cheb_hi > prm->cheb_lo, GMG_E_INVALID_ARG, "cheb range");
    GMG_REQUIRE(prm->eig_iters >= 1, GMG_E_INVALID_ARG, "eig_iters");
    GMG_REQUIRE(prm->coarse_solver == GMG_COARSE_CHOLESKY || prm->coarse_solver == GMG_COARSE_CHEBYSHEV,
                GMG_E_INVALID_ARG, "coarse_solver");
    auto h = std::make_unique<gmg_hierarchy>();
    h->prm = *prm;
    const bool rank_local = (prm->flags & GMG_RANK_LOCAL) != 0;
    const bool eig_key = rank_local || (prm->flags & GMG_EIG_KEY) != 0;
    const bool host_only = (prm->flags & GMG_HOST_ONLY) != 0;
    std::unique_ptr<gmg::Comm> comm;
    if (!host_only && prm->n_ranks > 1) {
      GMG_REQUIRE(prm->nccl_comm != nullptr, GMG_E_INVALID_ARG, "n_ranks > 1 needs a communicator");
      if (prm->device >= 0) {
        cudaError_t e = cudaSetDevice(prm->device);
        GMG_REQUIRE(e == cudaSuccess, GMG_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
      }
      if (prm->flags & GMG_HOST_RANKS) {
        auto* w = static_cast<gmg::HostWorld*>(prm->nccl_comm);
        GMG_REQUIRE(w->n == prm->n_ranks && w->rank == prm->rank, GMG_E_INVALID_ARG,
                    "host world rank/size != params");
        comm = std::make_unique<gmg::HostComm>(w);
      } else if (prm->flags & GMG_LOCAL_RANKS) {
        auto* w = static_cast<gmg::LocalWorld*>(prm->nccl_comm);
        GMG_REQUIRE(w->n == prm->n_ranks, GMG_E_INVALID_ARG, "local world size != n_ranks");
        comm = std::make_unique<gmg::ThreadComm>(w, prm->rank);
      } else {
        auto c = std::make_unique<gmg::NcclComm>(prm->nccl_comm);
        GMG_REQUIRE(c->size() == prm->n_ranks && c->rank() == prm->rank, GMG_E_INVALID_ARG,
                    "NCCL communicator rank/size != params");
        comm = std::move(c);
      }
    }
    GlobalSizes& z = h->sz;
    const gmg::Partition& P = p->p;
    z.dim = f->f.dim;
    z.k = prm->k;
    z.L = f->f.L;
    z.n_ranks = prm->n_ranks;
    const int nch = 1 << z.dim;
    for (int l = 0; l <= z.L; ++l) {
      const auto& c = P.levels[l];
      z.cells.push_back((gmg::i64)c.key.size());
      z.fams.push_back(l == 0 ? 0 : (gmg::i64)c.key.size() / nch);
      gmg::i64 nl = 0;
      for (auto x : c.leaf) nl += x ? 1 : 0;
      z.leaf_cells.push_back(nl);
    }
    if (!rank_local) {
      h->topo = gmg::make_topology(f->f, P, prm->k);
      h->local = gmg::make_local(f->f, P, h->topo, prm->rank, eig_key);
      const auto& T = h->topo;
      z.n_leaf_nodes = T.n_leaf_nodes;
      z.n_leaf_free = T.n_leaf;
      z.hanging = T.n_hanging;
      z.dirichlet = T.n_dirichlet;
      z.n0 = T.lv[0].n_dofs;
      for (int l = 0; l <= z.L; ++l) {
        z.dofs.push_back(T.lv[l].n_dofs);
        z.S.push_back(T.lv[l].nS);
        z.E.push_back(T.lv[l].nE);
        z.B.push_back(T.lv[l].nB);
      }
    } else {
      gmg::LocalCounts lc;
      h->local = gmg::make_local_direct(f->f, P, prm->k, prm->rank, true, &lc);
      // one sum over the ranks: [S | E | B | own_S | own_dofs] per level, 4 scalars,
      // and the owned leaf DoFs of every rank (slot r) for the leaf offsets
      const int nl = z.L + 1, R = prm->n_ranks;
      std::vector<double> v;
      for (auto* a : {&lc.S, &lc.E, &lc.B, &lc.own_S, &lc.own_dofs}) v.insert(v.end(), a->begin(), a->end());
      v.push_back(lc.leaf_nodes);
      v.push_back(lc.hanging);
      v.push_back(lc.dirichlet);
      v.push_back(lc.leaf_free);
      std::vector<double> leafc(R, 0.0);
      leafc[prm->rank] = (double)h->local.n_leaf_owned;
      v.insert(v.end(), leafc.begin(), leafc.end());
      const bool summed = comm != nullptr || R == 1;
      gmg::comm_allreduce_host(comm.get(), v);
      auto at = [&](int blk, int l) { return (gmg::i64)v[(size_t)blk * nl + l]; };
      for (int l = 0; l < nl; ++l) {
        z.S.push_back(summed ? at(0, l) : -1);
        z.E.push_back(summed ? at(1, l) : -1);
        z.B.push_back(summed ? at(2, l) : -1);
        z.dofs.push_back(summed ? at(4, l) : -1);
        h->local.lv[l].nS_global = summed ? at(3, l) : -1;
      }
      const size_t o = (size_t)5 * nl;
      if (summed) {
        z.n_leaf_nodes = (gmg::i64)v[o];
        z.hanging = (gmg::i64)v[o + 1];
        z.dirichlet = (gmg::i64)v[o + 2];
        z.n_leaf_free = (gmg::i64)v[o + 3];
        gmg::i64 first = 0;
        for (int q = 0; q < prm->rank; ++q) first += (gmg::i64)v[o + 4 + q];
        h->local.leaf_first = first;
        h->local.n_leaf_global = z.n_leaf_free;
      }
      z.n0 = summed ? at(4, 0) : h->local.lv[0].n_owned;
    }
    if (!host_only) {
      if (prm->coef_level2) gmg::attach_coefficients(h->local, f->f, P, prm->coef_level2);
      h->dev = gmg::device_create(h->local, *prm, std::move(comm), z.n0);
      // the device holds its own copies: drop the host tables (large for rank-local
      // runs of 125M DoFs per rank); keys, plans and counts stay for the exports
      for (auto& v : h->local.lv) {
        for (auto* t : {&v.cell_dofs, &v.xfer, &v.leaf_cells, &v.edge_fams, &v.gf_first}) {
          t->clear();
          t->shrink_to_fit();
        }
        for (auto* t : {&v.cls, &v.lam}) {
          t->clear();
          t->shrink_to_fit();
        }
        for (auto* t : {&v.eig_v, &v.cell_coef, &v.fam_coef, &v.cell_elem}) {
          t->clear();
          t->shrink_to_fit();
        }
        v.cell_global.clear();
        v.cell_global.shrink_to_fit();
      }
      h->local.leaf_local.clear();
      h->local.leaf_local.shrink_to_fit();
    }
    *out = h.release();
  });
}

gmg_status gmg_hierarchy_destroy(gmg_hierarchy* h) {
  return guard([&] { delete h; });
}

gmg_status gmg_leaf_layout(const gmg_hierarchy* h, int64_t* n_owned, int64_t* n_global, int64_t* first) {
  return guard([&] {
    NEED(h);
    if (n_owned) *n_owned = h->local.n_leaf_owned;
    if (n_global) *n_global = h->local.n_leaf_global;
    if (first) *first = h->local.leaf_first;
  });
}

gmg_status gmg_hierarchy_info(const gmg_hierarchy* h, gmg_info* o) {
  return guard([&] {
    NEED(h);
    NEED(o);
    std::memset(o, 0, sizeof *o);
    const GlobalSizes& z = h->sz;
    o->dim = z.dim;
    o->k = z.k;
    o->n_levels = z.L + 1;
    o->n_ranks = z.n_ranks;
    o->rank = h->prm.rank;
    o->n_leaf_nodes = z.n_leaf_nodes;
    o->n_leaf_free = z.n_leaf_free;
    o->n_leaf_hanging = z.hanging;
    o->n_leaf_dirichlet = z.dirichlet;
    o->n_owned = h->local.n_leaf_owned;
    o->first_owned = h->local.leaf_first;
    gmg::i64 mg = 0;
    for (int l = 0; l <= z.L && l < GMG_MAX_LEVELS; ++l) {
      o->level_dofs[l] = z.dofs[l];
      o->level_cells[l] = z.cells[l];
      o->level_families[l] = z.fams[l];
      o->level_S[l] = z.S[l];
      o->level_E[l] = z.E[l];
      o->level_B[l] = z.B[l];
      o->level_leaf_cells[l] = z.leaf_cells[l];
      o->level_r1[l] = h->dev ? gmg::device_level_r1(h->dev, l) : 0;
      o->level_gf[l] = h->dev ? gmg::device_level_gf(h->dev, l) : 0;
      // this rank's level vector (owned + ghosts), padded like the device segments (kernels.cuh VEC_PAD)
      mg += (h->local.lv[l].n_local() + 511) / 512 * 512;
    }
    o->mg_vector_len = h->dev ? gmg::device_mg_len(h->dev) : mg;
    o->small_levels = h->dev ? gmg::device_small_levels(h->dev) : 0;
  });
}

gmg_status gmg_export_level_dofs(const gmg_hierarchy* h, int level, int64_t* n, uint64_t* key, uint8_t* cls,
                                 int32_t* owner, int64_t* canonical) {
  return guard([&] {
    NEED(h);
    need_global(h);
    NEED(h);
    NEED(n);
    need_level(h, level);
    const auto& t = h->topo.lv[level];
    *n = t.n_dofs;
    for (gmg::i64 i = 0; i < t.n_dofs; ++i) {
      if (key) key[i] = t.dof_key[i];
      if (cls) cls[i] = t.dof_cls[i];
      if (owner) owner[i] = t.dof_owner[i];
      if (canonical) canonical[i] = t.dof_canon[i];
    }
  });
}

gmg_status gmg_export_leaf_dofs(const gmg_hierarchy* h, int64_t* n, uint64_t* key, int8_t* lambda, int32_t* owner,
                                int64_t* canonical) {
  return guard([&] {
    NEED(h);
    need_global(h);
    NEED(h);
    NEED(n);
    const auto& T = h->topo;
    *n = T.n_leaf;
    for (gmg::i64 i = 0; i < T.n_leaf; ++i) {
      if (key) key[i] = T.leaf_key[i];
      if (lambda) lambda[i] = T.leaf_lambda[i];
      if (owner) owner[i] = T.leaf_owner[i];
      if (canonical) canonical[i] = T.leaf_canon[i];
    }
  });
}

gmg_status gmg_export_rank_level(const gmg_hierarchy* h, int level, int64_t* first_owned, int64_t* n_owned,
                                 int64_t* n_ghost, int64_t* ghosts) {
  return guard([&] {
    NEED(h);
    need_level(h, level);
    need_global(h);
    const auto& v = h->local.lv[level];
    if (first_owned) *first_owned = v.first_owned;
    if (n_owned) *n_owned = v.n_owned;
    if (n_ghost) *n_ghost = v.n_ghost;
    if (ghosts)
      for (gmg::i64 i = 0; i < v.n_ghost; ++i) ghosts[i] = v.ghost_global[i];
  });
}

gmg_status gmg_nccl_get_unique_id(char id[128]) {
  return guard([&] {
    NEED(id);
    gmg::nccl_unique_id(id);
  });
}

gmg_status gmg_nccl_comm_init(const char id[128], int n_ranks, int rank, void** comm) {
  return guard([&] {
    NEED(id);
    NEED(comm);
    GMG_REQUIRE(n_ranks >= 1 && rank >= 0 && rank < n_ranks, GMG_E_INVALID_ARG, "rank / n_ranks");
    *comm = gmg::nccl_comm_init(id, n_ranks, rank);
  });
}

gmg_status gmg_nccl_comm_destroy(void* comm) {
  return guard([&] { gmg::nccl_comm_destroy(comm); });
}

gmg_status gmg_local_world_create(int n_ranks, void** world) {
  return guard([&] {
    NEED(world);
    GMG_REQUIRE(n_ranks >= 1 && n_ranks <= 64, GMG_E_INVALID_ARG, "n_ranks");
    *world = new gmg::LocalWorld(n_ranks);
  });
}

gmg_status gmg_local_world_destroy(void* world) {
  return guard([&] { delete static_cast<gmg::LocalWorld*>(world); });
}

gmg_status gmg_export_local_level(const gmg_hierarchy* h, int level, int64_t* n_owned, int64_t* n_ghost,
                                  uint64_t* owned_key, uint64_t* ghost_key, int32_t* ghost_owner, int32_t* n_peers,
                                  int32_t* peers, int64_t* send_off, int64_t* recv_off, int32_t* send_idx,
                                  int32_t* recv_idx) {
  return guard([&] {
    NEED(h);
    need_level(h, level);
    const auto& v = h->local.lv[level];
    if (n_owned) *n_owned = v.n_owned;
    if (n_ghost) *n_ghost = v.n_ghost;
    if (n_peers) *n_peers = (int32_t)v.peers.size();
    if (owned_key) std::copy(v.owned_key.begin(), v.owned_key.end(), owned_key);
    if (ghost_key) std::copy(v.ghost_key.begin(), v.ghost_key.end(), ghost_key);
    if (ghost_owner) std::copy(v.ghost_owner.begin(), v.ghost_owner.end(), ghost_owner);
    if (peers) std::copy(v.peers.begin(), v.peers.end(), peers);
    if (send_off) std::copy(v.send_off.begin(), v.send_off.end(), send_off);
    if (recv_off) std::copy(v.recv_off.begin(), v.recv_off.end(), recv_off);
    if (send_idx) std::copy(v.send_idx.begin(), v.send_idx.end(), send_idx);
    if (recv_idx) std::copy(v.recv_idx.begin(), v.recv_idx.end(), recv_idx);
  });
}

gmg_status gmg_export_local_tables(const gmg_hierarchy* h, int level, int64_t* n_cells, int64_t* n_fam,
                                   int32_t* cell_dofs, int32_t* xfer, uint8_t* cls, uint8_t* lam, double* eig_v,
                                   int64_t* cell_global) {
  return guard([&] {
    NEED(h);
    need_level(h, level);
    GMG_REQUIRE(h->dev == nullptr, GMG_E_STATE, "local tables are exported from GMG_HOST_ONLY hierarchies "
                                                "(device setup reorders them)");
    if (h->local.lv[level].eig_v.empty()) gmg::eig_start_from_keys(const_cast<gmg_hierarchy*>(h)->local);
    const auto& v = h->local.lv[level];
    if (n_cells) *n_cells = v.n_cells;
    if (n_fam) *n_fam = v.n_fam;
    if (cell_dofs) std::copy(v.cell_dofs.begin(), v.cell_dofs.end(), cell_dofs);
    if (xfer) std::copy(v.xfer.begin(), v.xfer.end(), xfer);
    if (cls) std::copy(v.cls.begin(), v.cls.end(), cls);
    if (lam) std::copy(v.lam.begin(), v.lam.end(), lam);
    if (eig_v) std::copy(v.eig_v.begin(), v.eig_v.end(), eig_v);
    if (cell_global) std::copy(v.cell_global.begin(), v.cell_global.end(), cell_global);
  });
}

gmg_status gmg_export_owned_leaf_keys(const gmg_hierarchy* h, int64_t* n, uint64_t* key, int8_t* lambda) {
  return guard([&] {
    NEED(h);
    NEED(n);
    *n = h->local.n_leaf_owned;
    if (key) std::copy(h->local.leaf_key.begin(), h->local.leaf_key.end(), key);
    if (lambda) std::copy(h->local.leaf_level.begin(), h->local.leaf_level.end(), lambda);
  });
}

gmg_status gmg_forest_count_nodes(const gmg_forest* f, int k, int64_t* n_nodes) {
  return guard([&] {
    NEED(f);
    NEED(n_nodes);
    *n_nodes = gmg::count_leaf_nodes(f->f, k);
  });
}

gmg_status gmg_profile_vcycle(gmg_hierarchy* h, const double* b, double* x, int n_rep, gmg_kernel_stat* out,
                              int max_out, int* n_out, void* stream) {
  return guard([&] {
    NEED(h);
    NEED(b);
    NEED(x);
    GMG_REQUIRE(n_rep >= 1 && max_out >= 0 && (out || max_out == 0), GMG_E_INVALID_ARG, "profile arguments");
    GMG_REQUIRE(h->dev != nullptr, GMG_E_STATE, "hierarchy has no device data (GMG_HOST_ONLY)");
    const int n = gmg::device_profile_vcycle(h->dev, b, x, n_rep, out, max_out, stream);
    if (n_out) *n_out = n;
  });
}

gmg_status gmg_host_world_create(const char* name, int n_ranks, int rank, size_t slot_bytes, void** world) {
  return guard([&] {
    NEED(name);
    NEED(world);
    *world = new gmg::HostWorld(name, n_ranks, rank, slot_bytes);
  });
}

gmg_status gmg_host_world_destroy(void* world) {
  return guard([&] { delete static_cast<gmg::HostWorld*>(world); });
}

gmg_status gmg_export_cell_dofs(const gmg_hierarchy* h, int level, int64_t* n_cells, int64_t* dofs) {
  return guard([&] {
    NEED(h);
    need_global(h);
    NEED(h);
    NEED(n_cells);
    need_level(h, level);
    const auto& t = h->topo.lv[level];
    *n_cells = t.n_cells;
    if (dofs)
      for (size_t i = 0; i < t.cell_dofs.size(); ++i) dofs[i] = t.cell_dofs[i];
  });
}

gmg_status gmg_vcycle(gmg_hierarchy* h, const double* b, double* x, void* s) {
  return guard([&] {
    NEED(h);
    NEED_LEAF(h, b);
    NEED_LEAF(h, x);
    GMG_REQUIRE(b != x || h->local.n_leaf_owned == 0, GMG_E_INVALID_ARG, "b and x must not alias");
    gmg::device_vcycle(need_dev(h), b, x, s);
  });
}

gmg_status gmg_solve_cg(gmg_hierarchy* h, const double* b, double* x, double rtol, int max_it, int* iters,
                        double* rel_res, void* s) {
  gmg_status st = GMG_OK;
  gmg_status g = guard([&] {
    NEED(h);
    NEED_LEAF(h, b);
    NEED_LEAF(h, x);
    GMG_REQUIRE(rtol >= 0 && max_it >= 1, GMG_E_INVALID_ARG, "rtol >= 0 and max_it >= 1 required");
    int rc = gmg::device_solve_cg(need_dev(h), b, x, rtol, max_it, iters, rel_res, s);
    if (rc) {
      g_err = "CG did not converge within max_it";
      st = GMG_E_NOT_CONVERGED;
    }
  });
  return g != GMG_OK ? g : st;
}

gmg_status gmg_rhs_constant(gmg_hierarchy* h, double f, double* b, void* s) {
  return guard([&] {
    NEED(h);
    NEED_LEAF(h, b);
    gmg::device_rhs_constant(need_dev(h), f, b, s);
  });
}

gmg_status gmg_level_apply(gmg_hierarchy* h, int level, const double* x, double* y, void* s) {
  return guard([&] {
    NEED(h);
    NEED(x);
    NEED(y);
    need_level(h, level);
    gmg::device_level_apply(need_dev(h), level, x, y, s);
  });
}

gmg_status gmg_level_apply_kernel(gmg_hierarchy* h, int level, const double* x, double* y, void* s) {
  return guard([&] {
    NEED(h);
    NEED(x);
    NEED(y);
    need_level(h, level);
    gmg::device_level_apply_kernel(need_dev(h), level, x, y, s);
  });
}

gmg_status gmg_level_apply_kernel_f32(gmg_hierarchy* h, int level, const float* x, float* y, void* s) {
  return guard([&] {
    NEED(h);
    NEED(x);
    NEED(y);
    need_level(h, level);
    gmg::device_level_apply_kernel_f32(need_dev(h), level, x, y, s);
  });
}

gmg_status gmg_restrict(gmg_hierarchy* h, int level, const double* r, double* dc, void* s) {
  return guard([&] {
    NEED(h);
    NEED(r);
    NEED(dc);
    need_level(h, level);
    GMG_REQUIRE(level >= 1, GMG_E_INVALID_ARG, "restriction needs level >= 1");
    gmg::device_restrict(need_dev(h), level, r, dc, s);
  });
}

gmg_status gmg_prolongate(gmg_hierarchy* h, int level, const double* xc, double* xf, void* s) {
  return guard([&] {
    NEED(h);
    NEED(xc);
    NEED(xf);
    need_level(h, level);
    GMG_REQUIRE(level >= 1, GMG_E_INVALID_ARG, "prolongation needs level >= 1");
    gmg::device_prolongate(need_dev(h), level, xc, xf, s);
  });
}

gmg_status gmg_leaf_apply(gmg_hierarchy* h, const double* u, double* v, void* s) {
  return guard([&] {
    NEED(h);
    NEED_LEAF(h, u);
    NEED_LEAF(h, v);
    gmg::device_leaf_apply(need_dev(h), u, v, s);
  });
}

gmg_status gmg_level_smooth(gmg_hierarchy* h, int level, const double* g, double* x, int x_is_zero, void* s) {
  return guard([&] {
    NEED(h);
    NEED(g);
    NEED(x);
    need_level(h, level);
    gmg::device_level_smooth(need_dev(h), level, g, x, x_is_zero, s);
  });
}

gmg_status gmg_level_diagonal(gmg_hierarchy* h, int level, double* diag, void* s) {
  return guard([&] {
    NEED(h);
    NEED(diag);
    need_level(h, level);
    gmg::device_level_diagonal(need_dev(h), level, diag, s);
  });
}

gmg_status gmg_get_coarse_chebyshev(const gmg_hierarchy* h, double* lo, double* hi, int* degree) {
  return guard([&] {
    NEED(h);
    NEED(lo);
    NEED(hi);
    NEED(degree);
    GMG_REQUIRE(h->dev != nullptr, GMG_E_STATE, "hierarchy has no device data (GMG_HOST_ONLY)");
    gmg::device_coarse_chebyshev(h->dev, lo, hi, degree);
  });
}

gmg_status gmg_get_eigen(const gmg_hierarchy* h, int level, double* lam) {
  return guard([&] {
    NEED(h);
    NEED(lam);
    need_level(h, level);
    GMG_REQUIRE(h->dev != nullptr, GMG_E_STATE, "no device data");
    *lam = gmg::device_get_eigen(h->dev, level);
  });
}

gmg_status gmg_set_eigen(gmg_hierarchy* h, int level, double lam) {
  return guard([&] {
    NEED(h);
    need_level(h, level);
    GMG_REQUIRE(h->dev != nullptr, GMG_E_STATE, "no device data");
    GMG_REQUIRE(level >= 1 && lam > 0 && std::isfinite(lam), GMG_E_INVALID_ARG, "lambda must be > 0 on level >= 1");
    gmg::device_set_eigen(h->dev, level, lam);
  });
}

gmg_status gmg_launch_count(const gmg_hierarchy* h, int64_t* count) {
  return guard([&] {
    NEED(h);
    NEED(count);
    *count = h->dev ? gmg::device_launches(h->dev) : 0;
  });
}

gmg_status gmg_launch_profile(const gmg_hierarchy* h, int64_t* pv, int64_t* pl) {
  return guard([&] {
    NEED(h);
    NEED(pv);
    NEED(pl);
    long long a = 0, b = 0;
    if (h->dev) gmg::device_launch_profile(h->dev, &a, &b);
    *pv = a;
    *pl = b;
  });
}

}  // extern "C"
