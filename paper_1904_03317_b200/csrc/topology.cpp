// Level DoF topology (host, integer): D_l, classes S/E/B, numbering, cell ->
// DoF tables, transfer ownership, lambda slots and the free leaf DoFs.
//
// Definitions (DESIGN.md notation): C_l = cells of level l; D_l = their
// Q_k nodes; B_l = D_l on the boundary; E_l = D_l \ B_l on the closure of a
// leaf of level < l; S_l = the rest.  lambda(n) = max{l : n in S_l}.
//
// Construction (independent of the oracle's definitions-by-search): every
// level-l cell (l >= 1) belongs to a family of 2^d siblings whose parent P is a
// refined level-(l-1) cell.  The (2k+1)^d nodes of a family patch are
// classified from the 3^d - 1 same-level neighbours of P: a neighbour outside
// the domain marks the shared patch nodes B, a neighbour that is a leaf (by
// 2:1 balance, the only coarser leaves touching C_l are of level l-1 and are
// neighbours of the parents) marks them E.
#include <numeric>

#include "patch.hpp"

namespace gmg {

Topology make_topology(const Forest& f, const Partition& p, int k) {
  GMG_REQUIRE(k == 1 || k == 2, GMG_E_INVALID_ARG, "k must be 1 or 2");
  Topology T;
  const int d = f.dim, L = f.L;
  T.dim = d;
  T.k = k;
  T.L = L;
  T.n_ranks = p.n_ranks;
  const i64 emax = std::max({f.ext[0], f.ext[1], f.ext[2]});
  const int cbits = bits_for((u64)(k * emax) << L);
  GMG_REQUIRE(cbits * d <= 64 && (d == 2 || cbits <= 21), GMG_E_DEPTH, "lattice keys exceed 64 bits");
  const int kbits = cbits * d;
  PatchTables pt(d, k);
  const int nn = pt.nn, np = pt.np, nch = pt.nch;
  T.lv.resize(L + 1);
  for (int l = 0; l <= L; ++l) {
    LevelTopo& t = T.lv[l];
    const LevelCells& cells = p.levels[l];
    t.level = l;
    t.n_cells = (i64)cells.key.size();
    for (i64 c = 0; c < t.n_cells; ++c)
      if (cells.leaf[c]) t.leaf_cells.push_back((i32)c);
    // ---------------- occurrences (key, id, flags, owner)
    i64 n_occ;
    std::vector<u64> okey, oid;
    std::vector<uint8_t> oflag;
    std::vector<i32> oown;
    if (l == 0) {
      n_occ = t.n_cells * nn;
      okey.resize(n_occ);
      oid.resize(n_occ);
      oflag.resize(n_occ);
      oown.resize(n_occ);
      for (i64 c = 0; c < t.n_cells; ++c) {
        Vec3 G = unmorton(d, cells.key[c]);
        for (int b = 0; b < nn; ++b) {
          Vec3 X{0, 0, 0};
          int r = b;
          for (int j = 0; j < d; ++j) {
            X[j] = ((i64)k * G[j] + r % (k + 1)) << L;
            r /= (k + 1);
          }
          i64 o = c * nn + b;
          okey[o] = morton(d, X);
          oid[o] = (u64)o;
          oflag[o] = (on_boundary(f, k, X) ? F_B : 0) | (cells.leaf[c] ? F_LEAF : 0);
          oown[o] = 0;   // coarse handoff: every level-0 DoF is owned by rank 0 (R25)
        }
      }
    } else {
      const LevelCells& par = p.levels[l - 1];
      for (i64 c = 0; c < (i64)par.key.size(); ++c)
        if (!par.leaf[c]) t.fam_parent.push_back((i32)c);
      t.n_fam = (i64)t.fam_parent.size();
      GMG_REQUIRE(t.n_fam * nch == t.n_cells, GMG_E_STATE, "level cells are not complete families");
      n_occ = t.n_fam * np;
      okey.resize(n_occ);
      oid.resize(n_occ);
      oflag.resize(n_occ);
      oown.resize(n_occ);
      for (i64 fi = 0; fi < t.n_fam; ++fi) {
        u64 pkey = par.key[t.fam_parent[fi]];
        for (int c = 0; c < nch; ++c)
          GMG_REQUIRE(cells.key[fi * nch + c] == ((pkey << d) | (u64)c), GMG_E_STATE,
                      "family children out of order");
        Vec3 G = unmorton(d, pkey);
        u32 outside = 0, leafn = 0;
        for (int o = 0; o < pt.ndir; ++o) {
          Vec3 off{o % 3 - 1, (o / 3) % 3 - 1, d == 3 ? o / 9 - 1 : 0};
          if (off[0] == 0 && off[1] == 0 && off[2] == 0) continue;
          Vec3 Q{G[0] + off[0], G[1] + off[1], G[2] + off[2]};
          if (!f.in_domain(l - 1, Q)) outside |= 1u << o;
          else if (!f.is_refined(l - 1, morton(d, Q))) leafn |= 1u << o;
        }
        for (int a = 0; a < np; ++a) {
          Vec3 X{0, 0, 0};
          for (int j = 0; j < d; ++j) X[j] = ((i64)2 * k * G[j] + pt.pa[a][j]) << (L - l);
          i64 o = fi * np + a;
          okey[o] = morton(d, X);
          oid[o] = (u64)o;
          uint8_t fl = 0;
          if (pt.dirmask[a] & outside) fl |= F_B;
          if (pt.dirmask[a] & leafn) fl |= F_EREG;
          for (int c = 0; c < nch; ++c)
            if ((pt.childmask[a] & (1u << c)) && cells.leaf[fi * nch + c]) fl |= F_LEAF;
          oflag[o] = fl;
          // DoF owner = min owner of the families whose patch contains the node
          // (R25); a family belongs to the owner of its cells (= its parent's owner
          // under the first-child rule; its own rank under per-level
          // partitioning, R29): the rank that computes a family owns at least one
          // DoF-containing family of each DoF it owns
          oown[o] = cells.owner[fi * nch];
        }
      }
    }
    radix_sort_pairs(okey, oid, kbits);
    // ---------------- unique nodes
    std::vector<i32> node_of_occ(n_occ);
    std::vector<u64> nkey;
    std::vector<uint8_t> nfl;
    std::vector<i32> nown;
    std::vector<i64> nfirst;
    for (i64 s = 0; s < n_occ;) {
      i64 e = s;
      uint8_t fl = 0;
      i32 own = INT32_MAX;
      while (e < n_occ && okey[e] == okey[s]) {
        i64 o = (i64)oid[e];
        fl |= oflag[o];
        own = std::min(own, oown[o]);
        node_of_occ[o] = (i32)nkey.size();
        ++e;
      }
      // transfer owner: the first family (SFC order) containing the node among
      // the families computed by the node's owner rank (R26)
      i64 first = INT64_MAX;
      for (i64 q = s; q < e; ++q)
        if (oown[oid[q]] == own) first = std::min(first, (i64)oid[q]);
      nkey.push_back(okey[s]);
      nfl.push_back(fl);
      nown.push_back(own);
      nfirst.push_back(first);
      s = e;
    }
    okey.clear(); okey.shrink_to_fit();
    oid.clear(); oid.shrink_to_fit();
    const i64 nnodes = (i64)nkey.size();
    // ---------------- counts (leaf nodes, hanging, Dirichlet)
    const i64 cstep = (i64)1 << (L - l + 1);   // coarse (l-1) node lattice spacing
    for (i64 r = 0; r < nnodes; ++r) {
      uint8_t fl = nfl[r];
      bool B = fl & F_B, Ereg = fl & F_EREG, inleaf = fl & F_LEAF;
      if (B) t.nB++;
      else if (Ereg) t.nE++;
      else t.nS++;
      if (!inleaf) continue;
      bool coarse = false;
      if (l > 0 && Ereg) {
        Vec3 X = unmorton(d, nkey[r]);
        coarse = true;
        for (int j = 0; j < d; ++j)
          if (X[j] % cstep) coarse = false;
      }
      if (Ereg && coarse) continue;          // counted on level l-1
      t.leaf_nodes++;
      if (B) t.dirichlet++;
      else if (Ereg) t.hanging++;
    }
    // ---------------- canonical and global numbering of S u E
    std::vector<i64> canon_of_node(nnodes, -1);
    i64 nd = 0;
    for (i64 r = 0; r < nnodes; ++r)
      if (!(nfl[r] & F_B)) canon_of_node[r] = nd++;
    t.n_dofs = nd;
    // counting sort by owner over canonical order
    const int P = p.n_ranks;
    std::vector<i64> cnt(P + 1, 0);
    for (i64 r = 0; r < nnodes; ++r)
      if (canon_of_node[r] >= 0) cnt[nown[r] + 1]++;
    for (int q = 0; q < P; ++q) cnt[q + 1] += cnt[q];
    std::vector<i64> glob_of_node(nnodes, -1);
    t.dof_key.resize(nd);
    t.dof_cls.resize(nd);
    t.dof_owner.resize(nd);
    t.dof_canon.resize(nd);
    t.canon_to_global.resize(nd);
    for (i64 r = 0; r < nnodes; ++r) {
      if (canon_of_node[r] < 0) continue;
      i64 g = cnt[nown[r]]++;
      glob_of_node[r] = g;
      t.dof_key[g] = nkey[r];
      t.dof_cls[g] = (nfl[r] & F_EREG) ? CLS_E : CLS_S;
      t.dof_owner[g] = nown[r];
      t.dof_canon[g] = canon_of_node[r];
      t.canon_to_global[canon_of_node[r]] = g;
    }
    // ---------------- cell -> dof table
    t.cell_dofs.resize((size_t)t.n_cells * nn);
    for (i64 c = 0; c < t.n_cells; ++c)
      for (int b = 0; b < nn; ++b) {
        i64 o = l == 0 ? c * nn + b : (c / nch) * np + pt.cell_to_patch[c % nch][b];
        t.cell_dofs[(size_t)c * nn + b] = (i32)glob_of_node[node_of_occ[o]];
      }
    // ---------------- family patch table with transfer ownership (the first
    // family containing a fine node owns it for restriction / prolongation)
    if (l > 0) {
      t.fam_dofs.resize((size_t)t.n_fam * np);
      std::vector<uint8_t> edge(t.n_fam, 0);
      for (i64 o = 0; o < n_occ; ++o) {
        const i64 r = node_of_occ[o];
        const i64 g = glob_of_node[r];
        if (g < 0) {
          t.fam_dofs[o] = -1;
        } else if (nfirst[r] == o) {
          t.fam_dofs[o] = (i32)g;
          if (nfl[r] & F_EREG) edge[o / np] = 1;
        } else {
          t.fam_dofs[o] = (i32)(-2 - g);
        }
      }
      for (i64 fi = 0; fi < t.n_fam; ++fi)
        if (edge[fi]) t.edge_fams.push_back((i32)fi);
    }
    t.dof_lam.assign(nd, 0);
  }
  // ---------------- lambda slots: S on l, not S on l+1
  for (int l = 0; l <= L; ++l) {
    LevelTopo& t = T.lv[l];
    std::vector<u64> upS;   // S keys of level l+1 on the level-l lattice (sorted)
    if (l < L) {
      const LevelTopo& u = T.lv[l + 1];
      const i64 step = (i64)1 << (L - l);
      for (i64 c = 0; c < u.n_dofs; ++c) {
        i64 g = u.canon_to_global[c];
        if (u.dof_cls[g] != CLS_S) continue;
        Vec3 X = unmorton(d, u.dof_key[g]);
        bool on = true;
        for (int j = 0; j < d; ++j)
          if (X[j] % step) on = false;
        if (on) upS.push_back(u.dof_key[g]);
      }
    }
    size_t q = 0;
    for (i64 c = 0; c < t.n_dofs; ++c) {
      i64 g = t.canon_to_global[c];
      u64 key = t.dof_key[g];
      while (q < upS.size() && upS[q] < key) ++q;
      bool up = q < upS.size() && upS[q] == key;
      t.dof_lam[g] = (t.dof_cls[g] == CLS_S && !up) ? 1 : 0;
    }
  }
  // ---------------- free leaf DoFs
  std::vector<u64> lkey, lidx;
  std::vector<int8_t> llam;
  std::vector<i32> lown;
  std::vector<i64> lglob;
  for (int l = 0; l <= L; ++l) {
    const LevelTopo& t = T.lv[l];
    for (i64 g = 0; g < t.n_dofs; ++g)
      if (t.dof_lam[g]) {
        lidx.push_back(lkey.size());
        lkey.push_back(t.dof_key[g]);
        llam.push_back((int8_t)l);
        lown.push_back(t.dof_owner[g]);
        lglob.push_back(g);
      }
    T.n_leaf_nodes += t.leaf_nodes;
    T.n_hanging += t.hanging;
    T.n_dirichlet += t.dirichlet;
  }
  radix_sort_pairs(lkey, lidx, kbits);
  const i64 nl = (i64)lkey.size();
  T.n_leaf = nl;
  const int P = p.n_ranks;
  std::vector<i64> cnt(P + 1, 0);
  for (i64 c = 0; c < nl; ++c) cnt[lown[lidx[c]] + 1]++;
  for (int q = 0; q < P; ++q) cnt[q + 1] += cnt[q];
  T.leaf_key.resize(nl);
  T.leaf_lambda.resize(nl);
  T.leaf_owner.resize(nl);
  T.leaf_canon.resize(nl);
  T.leaf_level_index.resize(nl);
  for (i64 c = 0; c < nl; ++c) {
    i64 o = (i64)lidx[c];
    i64 g = cnt[lown[o]]++;
    T.leaf_key[g] = lkey[c];
    T.leaf_lambda[g] = llam[o];
    T.leaf_owner[g] = lown[o];
    T.leaf_canon[g] = c;
    T.leaf_level_index[g] = lglob[o];
  }
  GMG_REQUIRE(T.n_leaf_nodes == T.n_leaf + T.n_hanging + T.n_dirichlet, GMG_E_STATE,
              "leaf node count mismatch");
  return T;
}

}  // namespace gmg
