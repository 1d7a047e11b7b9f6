// Forest of refinement trees, partition and level topology (host, integer).
#pragma once

#include "common.hpp"

namespace gmg {

// A forest over a brick of unit trees.  Cells are (level, G) with G the global
// brick coordinates on the level lattice; a cell's key is morton(G).
struct Forest {
  int dim = 2;
  std::vector<Vec3> trees;      // brick positions, z-ordered
  Vec3 ext{1, 1, 1};
  std::vector<uint8_t> occ;     // occupancy of brick positions
  int L = 0;                    // finest level
  std::vector<int8_t> level;    // leaves in SFC order
  std::vector<Vec3> gc;
  std::vector<std::vector<u64>> refined;  // per level: sorted keys of refined cells

  bool in_domain(int l, const Vec3& g) const {
    Vec3 t{0, 0, 0};
    for (int j = 0; j < dim; ++j) {
      if (g[j] < 0) return false;
      t[j] = g[j] >> l;
      if (t[j] >= ext[j]) return false;
    }
    return occ[(size_t)((t[2] * ext[1] + t[1]) * ext[0] + t[0])] != 0;
  }
  int tree_of(const Vec3& tpos) const;
  bool is_refined(int l, u64 key) const {
    if (l < 0 || l >= (int)refined.size()) return false;
    const auto& v = refined[l];
    auto it = std::lower_bound(v.begin(), v.end(), key);
    return it != v.end() && *it == key;
  }
  i64 n_leaves() const { return (i64)level.size(); }
};

Forest forest_from_refined(int dim, const std::vector<Vec3>& trees, std::vector<FlatSet>& R);
// Closure to 2:1 vertex balance: every refined cell of level >= 1 must have all
// its same-level neighbours (inside the domain) existing, i.e. their parents
// refined.  Processes the worklist of newly refined cells (level, key).
// Returns the number of cells refined by the closure.
i64 close_balance(int dim, const Forest& dom, std::vector<FlatSet>& R,
                  std::vector<std::pair<int, u64>>& work);
Forest forest_generate(const gmg_recipe& r);
i64 count_leaf_nodes(const Forest& f, int k);
Forest forest_sequence(int dim, gmg_sequence kind, int L);
Forest forest_create(int dim, int n_trees, const int32_t* tree_xyz, i64 n_leaves,
                     const int32_t* leaf_tree, const int8_t* leaf_level, const uint64_t* leaf_morton,
                     uint32_t flags);

// ------------------------------------------------------------------ partition
struct LevelCells {
  std::vector<u64> key;       // sorted
  std::vector<i32> owner;
  std::vector<uint8_t> leaf;
};

struct Partition {
  const Forest* f = nullptr;
  int n_ranks = 1;
  int mode = GMG_PARTITION_FIRST_CHILD;
  i64 coarse_cells = 0;        // levels 0.. with <= coarse_cells cells gathered on rank 0
  std::vector<i32> leaf_owner;
  std::vector<LevelCells> levels;
};

Partition make_partition(const Forest& f, int n_ranks, int mode = GMG_PARTITION_FIRST_CHILD, i64 coarse_cells = 0);
gmg_model partition_model(const Partition& p, i64 W0_override);

// ------------------------------------------------------------------ topology
enum : uint8_t { CLS_S = 0, CLS_E = 1 };

struct LevelTopo {
  int level = 0;
  i64 n_cells = 0;
  i64 n_fam = 0;
  std::vector<i32> fam_parent;     // index in C_{l-1}
  i64 n_dofs = 0;                  // |S u E|
  std::vector<u64> dof_key;        // global order
  std::vector<uint8_t> dof_cls;
  std::vector<i32> dof_owner;
  std::vector<i64> dof_canon;      // canonical (Morton) index of each global DoF
  std::vector<i64> canon_to_global;
  std::vector<uint8_t> dof_lam;    // lambda slot (S here, not S on l+1)
  std::vector<i32> cell_dofs;      // [n_cells][nn], global index or -1
  // [n_fam][(2k+1)^d] family patch -> level DoF: v >= 0 owned (transfers) by
  // this family, -1 Dirichlet, v <= -2 DoF -2-v owned by an earlier family
  std::vector<i32> fam_dofs;
  std::vector<i32> edge_fams;      // families owning >= 1 E patch node
  std::vector<i32> leaf_cells;     // cells of C_l that are leaves
  i64 nS = 0, nE = 0, nB = 0;
  i64 leaf_nodes = 0, hanging = 0, dirichlet = 0;
};

struct Topology {
  int dim = 2, k = 2, L = 0, n_ranks = 1;
  std::vector<LevelTopo> lv;
  // free leaf DoFs in global leaf order
  i64 n_leaf = 0;
  std::vector<u64> leaf_key;
  std::vector<int8_t> leaf_lambda;
  std::vector<i32> leaf_owner;
  std::vector<i64> leaf_canon;
  std::vector<i64> leaf_level_index;   // global level index at lambda
  i64 n_leaf_nodes = 0, n_hanging = 0, n_dirichlet = 0;
};

Topology make_topology(const Forest& f, const Partition& p, int k);

// ------------------------------------------------------------------ rank-local view
// Rank r computes the families whose parent it owns (first-child rule) and the
// level-0 cells it owns.  Its level vector = owned DoFs (a contiguous range of
// the global order) followed by ghost DoFs (owned elsewhere, needed by its
// families' patches or by the parents of its next-finer families), sorted by
// global index.  One exchange plan per level serves both directions:
//   import     owner -> ghost copies   (send_idx owned values, recv_idx ghosts)
//   export-add ghost -> owner, added    (reverse direction)
struct LocalLevel {
  int level = 0;
  i64 n_owned = 0, n_ghost = 0, first_owned = 0;
  std::vector<i64> ghost_global;           // sorted
  std::vector<int> peers;                  // ranks exchanged with (sorted)
  std::vector<i64> send_off, recv_off;     // [peers + 1]
  std::vector<i32> send_idx;               // local owned indices, grouped by peer
  std::vector<i32> recv_idx;               // local ghost indices, grouped by peer
  i64 n_cells = 0, n_fam = 0;
  std::vector<i32> cell_dofs;              // [n_cells][(k+1)^d] local index or -1
  // [n_fam][(2k+1)^d + (k+1)^d]: the family patch in local indices with the transfer-owner
  // encoding (v >= 0 this family owns the node for transfers, -2-v owned by another
  // family, -1 Dirichlet), then the parent's (k+1)^d level-(l-1) local DoFs
  std::vector<i32> xfer;
  std::vector<i32> leaf_cells, edge_fams;
  // complete grandfamilies (3D): local family index of the first of 8 consecutive
  // local families whose parents are the 8 children of one level-(l-2) cell
  std::vector<i32> gf_first;
  std::vector<uint8_t> cls, lam;           // per local DoF (ghosts: lam = 0)
  // rank-local builds (make_local_direct): finest-lattice Morton keys of the owned
  // DoFs and of the ghosts, and the ghosts' owners (ghost_global stays empty)
  std::vector<u64> owned_key, ghost_key;
  std::vector<i32> ghost_owner;
  std::vector<double> eig_v;               // eigen start vector on owned S DoFs
  i64 nS_global = 0;
  std::vector<i64> cell_global;            // global index (in C_l) of each local cell
  // variable coefficient (config 4; empty = a == 1), see coef.cpp
  std::vector<double> cell_coef;           // levels >= 2: a of each local cell
  std::vector<double> fam_coef;            // levels >= 3: a of each local family (one per family)
  std::vector<double> cell_elem;           // levels < 2: [n_cells][nn][nn] exact sub-box element matrices
  i64 n_local() const { return n_owned + n_ghost; }
};

struct LocalTopo {
  int rank = 0, n_ranks = 1, dim = 2, k = 2, L = 0;
  bool rank_local = false;                 // built by make_local_direct (no global numbering)
  std::vector<LocalLevel> lv;
  i64 n_leaf_owned = 0, leaf_first = 0, n_leaf_global = 0;
  std::vector<int8_t> leaf_level;          // per owned leaf DoF
  std::vector<i32> leaf_local;             // local index at its level
  std::vector<u64> leaf_key;               // finest-lattice key per owned leaf DoF
};

// eig_key: eigen start vector -5.5 + (level-lattice Morton key mod 12) on the
// owned S DoFs (reading R10b) instead of the canonical-rank pattern (R10)
LocalTopo make_local(const Forest& f, const Partition& p, const Topology& T, int rank, bool eig_key = false);

// Per-rank contributions to the global sizes of a rank-local build, summed over
// ranks by the caller (every node counted by exactly one rank).
struct LocalCounts {
  std::vector<double> S, E, B, own_S, own_dofs;   // per level
  double leaf_nodes = 0, hanging = 0, dirichlet = 0, leaf_free = 0;
  void resize(int L) {
    for (auto* v : {&S, &E, &B, &own_S, &own_dofs}) v->assign(L + 1, 0.0);
  }
};
LocalTopo make_local_direct(const Forest& f, const Partition& p, int k, int rank, bool eig_key,
                            LocalCounts* counts);
// the key-based eigen start vector (R10b) of every level whose eig_v is empty (rank-local
// builds store none); needs the local order (before the device reordering)
void eig_start_from_keys(LocalTopo& T);

// Piecewise-constant coefficient per level-2 cell (config 4): coef2[i] belongs to
// the i-th cell of C_2 in SFC order.  Fills the coefficient fields of every level.
void attach_coefficients(LocalTopo& Lt, const Forest& f, const Partition& p, const double* coef2);

}  // namespace gmg
