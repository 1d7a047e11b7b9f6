// Rank-local view of the level topology: owned/ghost DoFs, exchange plans,
// local cell / family / transfer tables ("ghost neighbors on each
// level ... information about parents/siblings is required for transfer
// operations"; computed redundantly on every rank without communication,
// P:611-613).
#include <numeric>

#include "forest.hpp"

namespace gmg {

static inline i64 decode_enc(i32 v) { return v >= 0 ? (i64)v : (v <= -2 ? -2 - (i64)v : -1); }

LocalTopo make_local(const Forest& f, const Partition& p, const Topology& T, int rank, bool eig_key) {
  const int d = T.dim, k = T.k, L = T.L, P = p.n_ranks;
  GMG_REQUIRE(rank >= 0 && rank < P, GMG_E_INVALID_ARG, "rank out of range");
  int nn = 1, np = 1;
  for (int j = 0; j < d; ++j) {
    nn *= k + 1;
    np *= 2 * k + 1;
  }
  const int nch = 1 << d;
  LocalTopo Lt;
  Lt.rank = rank;
  Lt.n_ranks = P;
  Lt.dim = d;
  Lt.k = k;
  Lt.L = L;
  Lt.lv.resize(L + 1);
  std::vector<std::vector<i64>> start(L + 1, std::vector<i64>(P + 1, 0));
  for (int l = 0; l <= L; ++l) {
    const LevelTopo& t = T.lv[l];
    for (i64 g = 0; g < t.n_dofs; ++g) start[l][t.dof_owner[g] + 1]++;
    for (int q = 0; q < P; ++q) start[l][q + 1] += start[l][q];
  }
  // the rank computing a family = the owner of its first child: under the first-child
  // rule the parent's owner; the other children may be owned elsewhere (ghost
  // children) and are still computed here.  Under per-level partitioning
  // (R29) families are kept whole and this is the family's rank.  Executed per-rank
  // work therefore follows family owners, not the cell owners the N_{l,p} model counts.
  auto fam_owner = [&](int l, i64 fi) { return p.levels[l].owner[fi * nch]; };
  // ---------------- ghost sets of every rank (needed DoFs owned elsewhere)
  std::vector<std::vector<std::vector<i64>>> ghosts(L + 1, std::vector<std::vector<i64>>(P));
  for (int l = 0; l <= L; ++l) {
    const LevelTopo& t = T.lv[l];
    auto need = [&](int q, i64 g) {
      if (g >= 0 && t.dof_owner[g] != q) ghosts[l][q].push_back(g);
    };
    if (l == 0) {
      for (i64 c = 0; c < t.n_cells; ++c)
        for (int b = 0; b < nn; ++b) need(p.levels[0].owner[c], t.cell_dofs[(size_t)c * nn + b]);
    } else {
      for (i64 fi = 0; fi < t.n_fam; ++fi) {
        const int q = fam_owner(l, fi);
        for (int a = 0; a < np; ++a) need(q, decode_enc(t.fam_dofs[(size_t)fi * np + a]));
      }
    }
    if (l < L) {   // parents of the next-finer families (prolongation / restriction targets)
      const LevelTopo& u = T.lv[l + 1];
      for (i64 fi = 0; fi < u.n_fam; ++fi) {
        const int q = fam_owner(l + 1, fi);
        const i64 c = u.fam_parent[fi];
        for (int b = 0; b < nn; ++b) need(q, t.cell_dofs[(size_t)c * nn + b]);
      }
    }
    for (int q = 0; q < P; ++q) {
      auto& v = ghosts[l][q];
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
    }
  }
  // ---------------- this rank
  std::vector<std::vector<i64>> cellg(L + 1);   // global cell index of each local cell
  std::vector<std::vector<i64>> famg(L + 1);    // global family index of each local family
  for (int l = 0; l <= L; ++l) {
    const LevelTopo& t = T.lv[l];
    LocalLevel& v = Lt.lv[l];
    v.level = l;
    v.first_owned = start[l][rank];
    v.n_owned = start[l][rank + 1] - start[l][rank];
    v.ghost_global = ghosts[l][rank];
    v.n_ghost = (i64)v.ghost_global.size();
    v.nS_global = t.nS;
    // plans: receive ghosts grouped by owner (global order is owner-major)
    std::vector<i64> rcount(P, 0), scount(P, 0);
    for (i64 g : v.ghost_global) rcount[t.dof_owner[g]]++;
    std::vector<std::vector<i32>> sidx(P);
    for (int q = 0; q < P; ++q) {
      if (q == rank) continue;
      for (i64 g : ghosts[l][q])
        if (t.dof_owner[g] == rank) sidx[q].push_back((i32)(g - v.first_owned));
      scount[q] = (i64)sidx[q].size();
    }
    v.send_off.push_back(0);
    v.recv_off.push_back(0);
    i64 gpos = 0;
    for (int q = 0; q < P; ++q) {
      if (rcount[q] == 0 && scount[q] == 0) {
        gpos += rcount[q];
        continue;
      }
      v.peers.push_back(q);
      for (i32 s : sidx[q]) v.send_idx.push_back(s);
      for (i64 c = 0; c < rcount[q]; ++c) v.recv_idx.push_back((i32)(v.n_owned + gpos + c));
      gpos += rcount[q];
      v.send_off.push_back((i64)v.send_idx.size());
      v.recv_off.push_back((i64)v.recv_idx.size());
    }
    // local cells / families
    if (l == 0) {
      for (i64 c = 0; c < t.n_cells; ++c)
        if (p.levels[0].owner[c] == rank) cellg[0].push_back(c);
    } else {
      for (i64 fi = 0; fi < t.n_fam; ++fi)
        if (fam_owner(l, fi) == rank) {
          famg[l].push_back(fi);
          for (int c = 0; c < nch; ++c) cellg[l].push_back(fi * nch + c);
        }
    }
    v.n_cells = (i64)cellg[l].size();
    v.cell_global = cellg[l];
    v.n_fam = (i64)famg[l].size();
    if (d == 3 && l >= 2) {
      // complete grandfamilies: 8 consecutive local families (SFC order) whose
      // parents are children 0..7 of one level-(l-2) cell
      const auto& pk = p.levels[l - 1].key;
      const i64 nf = v.n_fam;
      for (i64 lf = 0; lf + 7 < nf;) {
        const u64 k0 = pk[t.fam_parent[famg[l][lf]]];
        bool ok = (k0 & 7) == 0;
        for (int j = 1; ok && j < 8; ++j) ok = pk[t.fam_parent[famg[l][lf + j]]] == (k0 | (u64)j);
        if (ok) {
          v.gf_first.push_back((i32)lf);
          lf += 8;
        } else {
          ++lf;
        }
      }
    }
  }
  auto local_of = [&](int l, i64 g) -> i32 {
    if (g < 0) return -1;
    const LocalLevel& v = Lt.lv[l];
    if (g >= v.first_owned && g < v.first_owned + v.n_owned) return (i32)(g - v.first_owned);
    auto it = std::lower_bound(v.ghost_global.begin(), v.ghost_global.end(), g);
    GMG_REQUIRE(it != v.ghost_global.end() && *it == g, GMG_E_STATE, "DoF neither owned nor ghost");
    return (i32)(v.n_owned + (it - v.ghost_global.begin()));
  };
  for (int l = 0; l <= L; ++l) {
    const LevelTopo& t = T.lv[l];
    LocalLevel& v = Lt.lv[l];
    v.cell_dofs.resize((size_t)v.n_cells * nn);
    for (i64 c = 0; c < v.n_cells; ++c) {
      const i64 gc = cellg[l][c];
      for (int b = 0; b < nn; ++b) v.cell_dofs[(size_t)c * nn + b] = local_of(l, t.cell_dofs[(size_t)gc * nn + b]);
      if (p.levels[l].leaf[gc]) v.leaf_cells.push_back((i32)c);
    }
    const i64 nloc = v.n_local();
    v.cls.resize(nloc);
    v.lam.assign(nloc, 0);
    v.owned_key.resize(v.n_owned);
    v.ghost_key.resize(v.n_ghost);
    v.ghost_owner.resize(v.n_ghost);
    for (i64 i = 0; i < nloc; ++i) {
      const i64 g = i < v.n_owned ? v.first_owned + i : v.ghost_global[i - v.n_owned];
      v.cls[i] = t.dof_cls[g];
      if (i < v.n_owned) {
        v.lam[i] = t.dof_lam[g];
        v.owned_key[i] = t.dof_key[g];
      } else {
        v.ghost_key[i - v.n_owned] = t.dof_key[g];
        v.ghost_owner[i - v.n_owned] = t.dof_owner[g];
      }
    }
    // eigen start vector on owned S DoFs: -5.5 + (canonical S rank mod 12) (R10) or,
    // eig_key, -5.5 + (level-lattice Morton key mod 12) (R10b, the rank-local form)
    v.eig_v.assign(nloc, 0.0);
    if (eig_key) {
      for (i64 i = 0; i < v.n_owned; ++i) {
        const i64 g = v.first_owned + i;
        if (t.dof_cls[g] != CLS_S) continue;
        const Vec3 X = unmorton(d, t.dof_key[g]);
        Vec3 Y{0, 0, 0};
        for (int j = 0; j < d; ++j) Y[j] = X[j] >> (L - l);
        v.eig_v[i] = -5.5 + (double)(morton(d, Y) % 12);
      }
    } else {
      i64 cs = 0;
      for (i64 c = 0; c < t.n_dofs; ++c) {
        const i64 g = t.canon_to_global[c];
        if (t.dof_cls[g] != CLS_S) continue;
        if (g >= v.first_owned && g < v.first_owned + v.n_owned) v.eig_v[g - v.first_owned] = -5.5 + (double)(cs % 12);
        ++cs;
      }
    }
    if (l > 0) {
      const int row = np + nn;
      v.xfer.resize((size_t)v.n_fam * row);
      const LevelTopo& tc = T.lv[l - 1];
      for (i64 lf = 0; lf < v.n_fam; ++lf) {
        const i64 fi = famg[l][lf];
        bool edge = false;
        for (int a = 0; a < np; ++a) {
          const i32 e = t.fam_dofs[(size_t)fi * np + a];
          const i64 g = decode_enc(e);
          i32 enc = -1;
          if (g >= 0) {
            const i32 lg = local_of(l, g);
            enc = e >= 0 ? lg : -2 - lg;
            if (e >= 0) {
              GMG_REQUIRE(lg < v.n_owned, GMG_E_STATE, "transfer owner is not the DoF owner");
              if (t.dof_cls[g] == CLS_E) edge = true;
            }
          }
          v.xfer[(size_t)lf * row + a] = enc;
        }
        const i64 pc = t.fam_parent[fi];
        for (int j = 0; j < nn; ++j) v.xfer[(size_t)lf * row + np + j] = local_of(l - 1, tc.cell_dofs[(size_t)pc * nn + j]);
        if (edge) v.edge_fams.push_back((i32)lf);
      }
    }
  }
  // ---------------- owned free leaf DoFs (global leaf order is owner-major)
  Lt.n_leaf_global = T.n_leaf;
  i64 first = -1;
  for (i64 g = 0; g < T.n_leaf; ++g) {
    if (T.leaf_owner[g] != rank) continue;
    if (first < 0) first = g;
    const int l = T.leaf_lambda[g];
    Lt.leaf_level.push_back((int8_t)l);
    Lt.leaf_key.push_back(T.leaf_key[g]);
    Lt.leaf_local.push_back((i32)(T.leaf_level_index[g] - Lt.lv[l].first_owned));
    GMG_REQUIRE(Lt.leaf_local.back() >= 0 && Lt.leaf_local.back() < Lt.lv[l].n_owned, GMG_E_STATE,
                "leaf DoF not owned at its lambda level");
  }
  Lt.leaf_first = first < 0 ? 0 : first;
  Lt.n_leaf_owned = (i64)Lt.leaf_level.size();
  return Lt;
}

}  // namespace gmg
