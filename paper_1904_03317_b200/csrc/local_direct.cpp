// Rank-local level topology built WITHOUT the global level numbering: "it is
// advantageous for large computations if only the parts of the mesh relevant
// for the current processor are stored locally ... we need ghost neighbors on
// each level ... information about parents/siblings is required for transfer
// operations ... this ownership information is readily available without
// global communication" (§3.1).
//
// Produces the same LocalTopo as make_local (local.cpp) from the global
// Topology -- same owned/ghost sets and local order, exchange plans, cell /
// family / transfer tables, classes, lambda slots, leaf DoFs -- but touches only
// the families of this rank, the families whose parents contain the parents of
// this rank's next-finer families, and their vertex neighbours (the "halo").
// What needs other ranks' DoF counts (global leaf offset, global level sizes) is
// summed by the caller's allreduce afterwards (LocalCounts); the global DoF
// indices themselves are never formed (ghost_global stays empty; keys are kept).
//
// Why the halo suffices.  A node of a family F (level l) lies in the closure of
// F's parent P; every other family containing it has a parent touching P, i.e.
// one of P's 3^d - 1 vertex neighbours.  So owner (min computing rank of the
// families containing the node, R25), transfer owner (first such family of the
// owner, R26), class (B: some neighbour of P outside the domain shares it; E: a
// neighbour that is a leaf shares it) and the ranks that need the node (those
// computing a containing family; those computing the next-finer family of a
// containing refined cell) are all decided inside the halo.
#include <numeric>

#include "patch.hpp"

namespace gmg {

namespace {

struct Occ {
  u64 key;
  i64 fam;      // family index in C_l / nch (level >= 1) or cell index (level 0)
  int a;        // patch position (level >= 1) or local node (level 0)
};

}  // namespace

LocalTopo make_local_direct(const Forest& f, const Partition& p, int k, int rank, bool eig_key,
                            LocalCounts* counts) {
  GMG_REQUIRE(k == 1 || k == 2, GMG_E_INVALID_ARG, "k must be 1 or 2");
  const int d = f.dim, L = f.L, P = p.n_ranks;
  GMG_REQUIRE(rank >= 0 && rank < P, GMG_E_INVALID_ARG, "rank out of range");
  GMG_REQUIRE(eig_key, GMG_E_INVALID_ARG, "rank-local setup needs the key-based eigen start vector (R10b)");
  const i64 emax = std::max({f.ext[0], f.ext[1], f.ext[2]});
  const int cbits = bits_for((u64)(k * emax) << L);
  GMG_REQUIRE(cbits * d <= 64 && (d == 2 || cbits <= 21), GMG_E_DEPTH, "lattice keys exceed 64 bits");
  PatchTables pt(d, k);
  const int nn = pt.nn, np = pt.np, nch = pt.nch;
  LocalTopo Lt;
  Lt.rank = rank;
  Lt.n_ranks = P;
  Lt.dim = d;
  Lt.k = k;
  Lt.L = L;
  Lt.rank_local = true;
  Lt.lv.resize(L + 1);
  LocalCounts cnt;
  cnt.resize(L);

  // ---------------- helpers over the global partition (cells of every level, SFC order)
  auto nfam_of = [&](int l) -> i64 { return l == 0 ? 0 : (i64)p.levels[l].key.size() / nch; };
  auto comp = [&](int l, i64 fi) -> int { return p.levels[l].owner[(size_t)fi * nch]; };   // computing rank
  auto cell_index = [&](int l, u64 key) -> i64 {
    const auto& ks = p.levels[l].key;
    auto it = std::lower_bound(ks.begin(), ks.end(), key);
    return (it != ks.end() && *it == key) ? (i64)(it - ks.begin()) : -1;
  };
  // family (level l >= 1) of the children of level-(l-1) cell `pkey` (-1: not refined)
  auto fam_of_parent = [&](int l, u64 pkey) -> i64 {
    if (l > L) return -1;
    const i64 c = cell_index(l, pkey << d);
    return c < 0 ? -1 : c / nch;
  };
  auto parent_key = [&](int l, i64 fi) -> u64 { return p.levels[l].key[(size_t)fi * nch] >> d; };
  auto node_X = [&](int l, u64 pkey, int a) {   // finest-lattice coordinates of patch node a
    const Vec3 G = unmorton(d, pkey);
    Vec3 X{0, 0, 0};
    for (int j = 0; j < d; ++j) X[j] = ((i64)2 * k * G[j] + pt.pa[a][j]) << (L - l);
    return X;
  };

  // ---------------- families computed here, per level
  std::vector<std::vector<i64>> mine(L + 1);
  for (int l = 1; l <= L; ++l)
    for (i64 fi = 0; fi < nfam_of(l); ++fi)
      if (comp(l, fi) == rank) mine[l].push_back(fi);
  std::vector<i64> mine0;
  for (i64 c = 0; c < (i64)p.levels[0].key.size(); ++c)
    if (p.levels[0].owner[c] == rank) mine0.push_back(c);

  // per level: local index of every node this rank needs (by key), for the xfer
  // rows of the next level
  std::vector<std::vector<u64>> owned_keys(L + 1), ghost_keys(L + 1);
  std::vector<std::vector<std::pair<u64, i32>>> keymap(L + 1);   // key -> local index

  for (int l = 0; l <= L; ++l) {
    LocalLevel& v = Lt.lv[l];
    v.level = l;
    v.first_owned = -1;
    // ---------------- occurrences of the halo
    std::vector<Occ> occ;
    // needed: (key) of the nodes this rank needs
    std::vector<u64> need;
    if (l == 0) {
      const auto& c0 = p.levels[0];
      for (i64 c = 0; c < (i64)c0.key.size(); ++c) {
        const Vec3 G = unmorton(d, c0.key[c]);
        for (int b = 0; b < nn; ++b) {
          Vec3 X{0, 0, 0};
          int r = b;
          for (int j = 0; j < d; ++j) {
            X[j] = ((i64)k * G[j] + r % (k + 1)) << L;
            r /= (k + 1);
          }
          occ.push_back({morton(d, X), c, b});
        }
      }
      std::vector<char> needc(c0.key.size(), 0);
      for (i64 c : mine0) needc[c] = 1;
      if (L >= 1)
        for (i64 fi : mine[1]) needc[cell_index(0, parent_key(1, fi))] = 1;
      for (const Occ& o : occ)
        if (needc[o.fam]) need.push_back(o.key);
    } else {
      // families whose parents' nodes or patches this rank needs
      std::vector<i64> needfam = mine[l];
      std::vector<std::pair<i64, int>> needcell;   // (family, child) parents of next-level families
      if (l < L)
        for (i64 fi1 : mine[l + 1]) {
          const u64 pk = parent_key(l + 1, fi1);                 // a level-l cell
          const i64 c = cell_index(l, pk);
          needfam.push_back(c / nch);
          needcell.push_back({c / nch, (int)(c % nch)});
        }
      std::sort(needfam.begin(), needfam.end());
      needfam.erase(std::unique(needfam.begin(), needfam.end()), needfam.end());
      // halo: families whose parent is a vertex neighbour of a needed family's parent
      std::vector<i64> halo;
      for (i64 fi : needfam) {
        const Vec3 G = unmorton(d, parent_key(l, fi));
        for (int o = 0; o < pt.ndir; ++o) {
          const Vec3 Q{G[0] + o % 3 - 1, G[1] + (o / 3) % 3 - 1, d == 3 ? G[2] + o / 9 - 1 : 0};
          if (!f.in_domain(l - 1, Q)) continue;
          const i64 g = fam_of_parent(l, morton(d, Q));
          if (g >= 0) halo.push_back(g);
        }
      }
      std::sort(halo.begin(), halo.end());
      halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
      occ.reserve(halo.size() * np);
      for (i64 fi : halo) {
        const u64 pk = parent_key(l, fi);
        for (int a = 0; a < np; ++a) occ.push_back({morton(d, node_X(l, pk, a)), fi, a});
      }
      for (i64 fi : mine[l]) {
        const u64 pk = parent_key(l, fi);
        for (int a = 0; a < np; ++a) need.push_back(morton(d, node_X(l, pk, a)));
      }
      for (auto& fc : needcell) {
        const u64 pk = parent_key(l, fc.first);
        for (int b = 0; b < nn; ++b) need.push_back(morton(d, node_X(l, pk, pt.cell_to_patch[fc.second][b])));
      }
    }
    std::sort(occ.begin(), occ.end(), [](const Occ& a, const Occ& b) {
      return a.key != b.key ? a.key < b.key : (a.fam != b.fam ? a.fam < b.fam : a.a < b.a);
    });
    std::sort(need.begin(), need.end());
    need.erase(std::unique(need.begin(), need.end()), need.end());
    // ---------------- unique halo nodes: flags, owner, transfer owner
    struct Node {
      u64 key;
      uint8_t fl;
      int owner;
      i64 tfam;     // transfer-owner family (level >= 1)
      i64 o0, o1;   // occurrence range
    };
    std::vector<Node> nodes;
    for (size_t s = 0; s < occ.size();) {
      size_t e = s;
      Node nd{occ[s].key, 0, INT32_MAX, INT64_MAX, (i64)s, 0};
      while (e < occ.size() && occ[e].key == occ[s].key) ++e;
      nd.o1 = (i64)e;
      for (size_t q = s; q < e; ++q) {
        const Occ& o = occ[q];
        if (l == 0) {
          nd.owner = 0;                                          // coarse handoff (R25)
          if (p.levels[0].leaf[o.fam]) nd.fl |= F_LEAF;
          continue;
        }
        const int cr = comp(l, o.fam);
        nd.owner = std::min(nd.owner, cr);
        for (int c = 0; c < nch; ++c)
          if ((pt.childmask[o.a] & (1u << c)) && p.levels[l].leaf[(size_t)o.fam * nch + c]) nd.fl |= F_LEAF;
      }
      if (l == 0) {
        if (on_boundary(f, k, unmorton(d, nd.key))) nd.fl |= F_B;
      } else {
        for (size_t q = s; q < e; ++q) {
          const Occ& o = occ[q];
          if (comp(l, o.fam) == nd.owner) nd.tfam = std::min(nd.tfam, o.fam);
        }
        // class from the parent's neighbours (as topology.cpp), any occurrence decides
        const Occ& o = occ[s];
        const Vec3 G = unmorton(d, parent_key(l, o.fam));
        for (int dd = 0; dd < pt.ndir; ++dd) {
          if (!(pt.dirmask[o.a] & (1u << dd))) continue;
          const Vec3 Q{G[0] + dd % 3 - 1, G[1] + (dd / 3) % 3 - 1, d == 3 ? G[2] + dd / 9 - 1 : 0};
          if (!f.in_domain(l - 1, Q)) nd.fl |= F_B;
          else if (!f.is_refined(l - 1, morton(d, Q))) nd.fl |= F_EREG;
        }
      }
      nodes.push_back(nd);
      s = e;
    }
    auto node_of = [&](u64 key) -> i64 {
      auto it = std::lower_bound(nodes.begin(), nodes.end(), key, [](const Node& a, u64 kk) { return a.key < kk; });
      GMG_REQUIRE(it != nodes.end() && it->key == key, GMG_E_STATE, "node outside the halo");
      return (i64)(it - nodes.begin());
    };
    // ---------------- counts (each node counted by its owner; B nodes by the min computing rank)
    {
      const i64 cstep = (i64)1 << (L - l + 1);
      for (const Node& nd : nodes) {
        // only nodes whose containing families are complete in the halo: the owner's
        // own nodes (owner == rank => the node is in one of this rank's families)
        if (nd.owner != rank) continue;
        if (l > 0) {
          bool in_mine = false;
          for (i64 q = nd.o0; q < nd.o1 && !in_mine; ++q) in_mine = comp(l, occ[q].fam) == rank;
          if (!in_mine) continue;
        } else if (rank != 0) {
          continue;
        }
        const bool B = nd.fl & F_B, E = nd.fl & F_EREG, inleaf = nd.fl & F_LEAF;
        if (B) cnt.B[l]++;
        else if (E) cnt.E[l]++;
        else cnt.S[l]++;
        if (!inleaf) continue;
        bool coarse = false;
        if (l > 0 && E) {
          const Vec3 X = unmorton(d, nd.key);
          coarse = true;
          for (int j = 0; j < d; ++j)
            if (X[j] % cstep) coarse = false;
        }
        if (E && coarse) continue;
        cnt.leaf_nodes++;
        if (B) cnt.dirichlet++;
        else if (E) cnt.hanging++;
      }
    }
    // ---------------- owned and ghost DoFs (local order = global order restricted)
    std::vector<i64> owned, ghosts;       // node indices
    if (l == 0 && rank == 0) {
      for (i64 i = 0; i < (i64)nodes.size(); ++i)
        if (!(nodes[i].fl & F_B)) owned.push_back(i);
    }
    for (u64 kk : need) {
      const i64 i = node_of(kk);
      if (nodes[i].fl & F_B) continue;
      if (nodes[i].owner == rank) {
        if (l > 0) owned.push_back(i);
      } else {
        ghosts.push_back(i);
      }
    }
    std::sort(owned.begin(), owned.end());
    owned.erase(std::unique(owned.begin(), owned.end()), owned.end());
    std::sort(ghosts.begin(), ghosts.end(), [&](i64 a, i64 b) {
      return nodes[a].owner != nodes[b].owner ? nodes[a].owner < nodes[b].owner : nodes[a].key < nodes[b].key;
    });
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    v.n_owned = (i64)owned.size();
    v.n_ghost = (i64)ghosts.size();
    const i64 nloc = v.n_local();
    std::vector<i32> local(nodes.size(), -1);
    for (i64 i = 0; i < v.n_owned; ++i) local[owned[i]] = (i32)i;
    for (i64 i = 0; i < v.n_ghost; ++i) local[ghosts[i]] = (i32)(v.n_owned + i);
    owned_keys[l].resize(v.n_owned);
    ghost_keys[l].resize(v.n_ghost);
    v.ghost_owner.resize(v.n_ghost);
    for (i64 i = 0; i < v.n_owned; ++i) owned_keys[l][i] = nodes[owned[i]].key;
    for (i64 i = 0; i < v.n_ghost; ++i) {
      ghost_keys[l][i] = nodes[ghosts[i]].key;
      v.ghost_owner[i] = nodes[ghosts[i]].owner;
    }
    v.owned_key = owned_keys[l];
    v.ghost_key = ghost_keys[l];
    keymap[l].reserve(nloc);
    for (i64 i = 0; i < v.n_owned; ++i) keymap[l].push_back({owned_keys[l][i], (i32)i});
    for (i64 i = 0; i < v.n_ghost; ++i) keymap[l].push_back({ghost_keys[l][i], (i32)(v.n_owned + i)});
    std::sort(keymap[l].begin(), keymap[l].end());
    // ---------------- exchange plan: who needs each owned DoF
    std::vector<std::vector<i32>> sidx(P);
    if (l == 0) {
      if (rank == 0) {
        // rank q needs the nodes of its level-0 cells and of the parents of its level-1 families
        std::vector<std::vector<char>> needq(P, std::vector<char>(p.levels[0].key.size(), 0));
        for (i64 c = 0; c < (i64)p.levels[0].key.size(); ++c) needq[p.levels[0].owner[c]][c] = 1;
        if (L >= 1)
          for (i64 fi = 0; fi < nfam_of(1); ++fi) needq[comp(1, fi)][cell_index(0, parent_key(1, fi))] = 1;
        for (int q = 1; q < P; ++q) {
          std::vector<i64> ns;
          for (const Occ& o : occ)
            if (needq[q][o.fam]) ns.push_back(node_of(o.key));
          std::sort(ns.begin(), ns.end());
          ns.erase(std::unique(ns.begin(), ns.end()), ns.end());
          for (i64 i : ns)
            if (!(nodes[i].fl & F_B)) sidx[q].push_back(local[i]);
        }
      }
    } else {
      for (i64 oi = 0; oi < v.n_owned; ++oi) {
        const Node& nd = nodes[owned[oi]];
        std::vector<int> qs;
        for (i64 q = nd.o0; q < nd.o1; ++q) {
          const Occ& o = occ[q];
          qs.push_back(comp(l, o.fam));                        // operator: a containing family
          for (int c = 0; c < nch; ++c) {                        // transfer: next-finer family of a refined cell
            if (!(pt.childmask[o.a] & (1u << c))) continue;
            if (p.levels[l].leaf[(size_t)o.fam * nch + c]) continue;
            const i64 f1 = fam_of_parent(l + 1, p.levels[l].key[(size_t)o.fam * nch + c]);
            if (f1 >= 0) qs.push_back(comp(l + 1, f1));
          }
        }
        std::sort(qs.begin(), qs.end());
        qs.erase(std::unique(qs.begin(), qs.end()), qs.end());
        for (int q : qs)
          if (q != rank) sidx[q].push_back((i32)oi);
      }
    }
    std::vector<i64> rcount(P, 0);
    for (i64 i = 0; i < v.n_ghost; ++i) rcount[v.ghost_owner[i]]++;
    v.send_off.push_back(0);
    v.recv_off.push_back(0);
    i64 gpos = 0;
    for (int q = 0; q < P; ++q) {
      if (rcount[q] == 0 && sidx[q].empty()) continue;
      v.peers.push_back(q);
      for (i32 s : sidx[q]) v.send_idx.push_back(s);
      for (i64 c = 0; c < rcount[q]; ++c) v.recv_idx.push_back((i32)(v.n_owned + gpos + c));
      gpos += rcount[q];
      v.send_off.push_back((i64)v.send_idx.size());
      v.recv_off.push_back((i64)v.recv_idx.size());
    }
    // ---------------- local cells / families and their tables
    if (l == 0) {
      for (i64 c : mine0) v.cell_global.push_back(c);
    } else {
      for (i64 fi : mine[l])
        for (int c = 0; c < nch; ++c) v.cell_global.push_back(fi * nch + c);
    }
    v.n_cells = (i64)v.cell_global.size();
    v.n_fam = l == 0 ? 0 : (i64)mine[l].size();
    v.cell_dofs.resize((size_t)v.n_cells * nn);
    for (i64 c = 0; c < v.n_cells; ++c) {
      const i64 gc = v.cell_global[c];
      for (int b = 0; b < nn; ++b) {
        u64 key;
        if (l == 0) {
          const Vec3 G = unmorton(d, p.levels[0].key[gc]);
          Vec3 X{0, 0, 0};
          int r = b;
          for (int j = 0; j < d; ++j) {
            X[j] = ((i64)k * G[j] + r % (k + 1)) << L;
            r /= (k + 1);
          }
          key = morton(d, X);
        } else {
          key = morton(d, node_X(l, parent_key(l, gc / nch), pt.cell_to_patch[gc % nch][b]));
        }
        const i64 i = node_of(key);
        v.cell_dofs[(size_t)c * nn + b] = (nodes[i].fl & F_B) ? -1 : local[i];
      }
      if (p.levels[l].leaf[gc]) v.leaf_cells.push_back((i32)c);
    }
    v.cls.resize(nloc);
    v.lam.assign(nloc, 0);
    v.eig_v.assign(nloc, 0.0);
    auto fill_node = [&](i64 li, i64 i) {
      const Node& nd = nodes[i];
      v.cls[li] = (nd.fl & F_EREG) ? CLS_E : CLS_S;
      if (li >= v.n_owned || v.cls[li] != CLS_S) return;
      // lambda slot: S here and some in-domain level-l cell containing the node is a leaf
      const Vec3 X = unmorton(d, nd.key);
      const i64 s = (i64)k << (L - l);
      bool up = true;
      for (int c = 0; c < (1 << d) && up; ++c) {
        Vec3 Q{0, 0, 0};
        for (int j = 0; j < d; ++j) Q[j] = ((c >> j) & 1) ? X[j] / s : (X[j] - 1) / s - ((X[j] - 1) < 0 ? 1 : 0);
        bool neg = false;
        for (int j = 0; j < d; ++j) neg |= Q[j] < 0;
        if (neg || !f.in_domain(l, Q)) continue;
        if (!f.is_refined(l, morton(d, Q))) up = false;
      }
      v.lam[li] = up ? 0 : 1;
      // eigen start vector, key-based (R10b): -5.5 + (level-lattice Morton key mod 12)
      Vec3 Y{0, 0, 0};
      for (int j = 0; j < d; ++j) Y[j] = X[j] >> (L - l);
      v.eig_v[li] = -5.5 + (double)(morton(d, Y) % 12);
    };
    for (i64 i = 0; i < v.n_owned; ++i) fill_node(i, owned[i]);
    for (i64 i = 0; i < v.n_ghost; ++i) fill_node(v.n_owned + i, ghosts[i]);
    for (i64 i = 0; i < v.n_owned; ++i)
      if (v.cls[i] == CLS_S) cnt.own_S[l]++;
    if (l > 0) {
      const int row = np + nn;
      v.fam_dofs.resize((size_t)v.n_fam * np);
      v.xfer.resize((size_t)v.n_fam * row);
      const auto& km = keymap[l - 1];
      auto local_coarse = [&](u64 key) -> i32 {   // level-(l-1) local index of a node (-1: Dirichlet / absent)
        auto it = std::lower_bound(km.begin(), km.end(), std::make_pair(key, (i32)INT32_MIN));
        return (it != km.end() && it->first == key) ? it->second : -1;
      };
      for (i64 lf = 0; lf < v.n_fam; ++lf) {
        const i64 fi = mine[l][lf];
        const u64 pk = parent_key(l, fi);
        bool edge = false;
        for (int a = 0; a < np; ++a) {
          const i64 i = node_of(morton(d, node_X(l, pk, a)));
          i32 enc = -1;
          if (!(nodes[i].fl & F_B)) {
            const i32 lg = local[i];
            GMG_REQUIRE(lg >= 0, GMG_E_STATE, "patch node without a local index");
            const bool towner = nodes[i].tfam == fi;
            enc = towner ? lg : -2 - lg;
            if (towner) {
              GMG_REQUIRE(lg < v.n_owned, GMG_E_STATE, "transfer owner is not the DoF owner");
              if (nodes[i].fl & F_EREG) edge = true;
            }
          }
          v.fam_dofs[(size_t)lf * np + a] = enc;
          v.xfer[(size_t)lf * row + a] = enc;
        }
        // the parent's (k+1)^d nodes on level l-1
        const i64 pc = cell_index(l - 1, pk);
        for (int b = 0; b < nn; ++b) {
          u64 key;
          if (l - 1 == 0) {
            const Vec3 G = unmorton(d, pk);
            Vec3 X{0, 0, 0};
            int r = b;
            for (int j = 0; j < d; ++j) {
              X[j] = ((i64)k * G[j] + r % (k + 1)) << L;
              r /= (k + 1);
            }
            key = morton(d, X);
          } else {
            const int child = (int)(pc % nch);
            key = morton(d, node_X(l - 1, parent_key(l - 1, pc / nch), pt.cell_to_patch[child][b]));
          }
          const i32 lc = local_coarse(key);
          v.xfer[(size_t)lf * row + np + b] = lc;
        }
        if (edge) v.edge_fams.push_back((i32)lf);
      }
      // complete grandfamilies (as make_local)
      if (d == 3 && l >= 2) {
        const auto& pkk = p.levels[l - 1].key;
        for (i64 lf = 0; lf + 7 < v.n_fam;) {
          const u64 k0 = pkk[cell_index(l - 1, parent_key(l, mine[l][lf]))];
          bool ok = (k0 & 7) == 0;
          for (int j = 1; ok && j < 8; ++j) ok = parent_key(l, mine[l][lf + j]) == (k0 | (u64)j);
          if (ok) {
            v.gf_first.push_back((i32)lf);
            lf += 8;
          } else {
            ++lf;
          }
        }
      }
    }
    // ---------------- owned free leaf DoFs of this level
    for (i64 i = 0; i < v.n_owned; ++i)
      if (v.lam[i]) Lt.leaf_tmp.push_back({owned_keys[l][i], (int8_t)l, i});
    cnt.own_dofs[l] = v.n_owned;
  }
  // leaf order (owner, key): this rank's leaf DoFs by key
  std::sort(Lt.leaf_tmp.begin(), Lt.leaf_tmp.end(),
            [](const LocalTopo::LeafRec& a, const LocalTopo::LeafRec& b) { return a.key < b.key; });
  for (const auto& r : Lt.leaf_tmp) {
    Lt.leaf_level.push_back(r.level);
    Lt.leaf_local.push_back(r.local);
    Lt.leaf_key.push_back(r.key);
  }
  Lt.leaf_tmp.clear();
  Lt.n_leaf_owned = (i64)Lt.leaf_level.size();
  Lt.leaf_first = -1;          // set from the other ranks' counts (LocalCounts)
  Lt.n_leaf_global = -1;
  cnt.leaf_free = Lt.n_leaf_owned;
  if (counts) *counts = cnt;
  return Lt;
}

}  // namespace gmg
