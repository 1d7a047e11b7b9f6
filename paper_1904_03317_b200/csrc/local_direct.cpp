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
// the families of this rank, the families whose cells are parents of this
// rank's next-finer families, and their vertex neighbours (the "halo").  What
// needs other ranks' DoF counts (global leaf offset, global level sizes) is
// summed by the caller afterwards (LocalCounts); global DoF indices are never
// formed (ghost_global stays empty; keys are kept).
//
// Why the halo suffices.  A node of a family F (level l) lies in the closure of
// F's parent P; every other family containing it has a parent touching P, i.e.
// one of P's 3^d - 1 vertex neighbours.  So owner (min computing rank of the
// families containing the node, R25), transfer owner (first such family of the
// owner, R26), class (B: a neighbour of P outside the domain shares it; E: a
// neighbour that is a leaf shares it), lambda (a containing level-l cell is a
// leaf) and the ranks that need the node (those computing a containing family;
// those computing the next-finer family of a containing refined cell) are all
// decided inside the halo.  Construction as topology.cpp: occurrences (key,
// halo family, patch position) radix-sorted by key, one pass over equal keys.
#include <cstdlib>
#include <numeric>

#include "patch.hpp"

namespace gmg {

namespace {

// LSD radix sort of (64-bit key, 32-bit value) pairs by key; stable.
void radix_sort_pairs32(std::vector<u64>& key, std::vector<u32>& val, int key_bits) {
  const size_t n = key.size();
  std::vector<u64> k2(n);
  std::vector<u32> v2(n);
  const int RB = 11, R = 1 << RB;
  std::vector<size_t> cnt(R);
  for (int shift = 0; shift < key_bits; shift += RB) {
    std::fill(cnt.begin(), cnt.end(), 0);
    for (size_t i = 0; i < n; ++i) cnt[(key[i] >> shift) & (R - 1)]++;
    size_t s = 0;
    for (int b = 0; b < R; ++b) {
      size_t c = cnt[b];
      cnt[b] = s;
      s += c;
    }
    for (size_t i = 0; i < n; ++i) {
      const size_t d = cnt[(key[i] >> shift) & (R - 1)]++;
      k2[d] = key[i];
      v2[d] = val[i];
    }
    key.swap(k2);
    val.swap(v2);
  }
}

// per level: what the next level needs from this one
struct LevelKeep {
  std::vector<i64> halo;          // halo families (level >= 1) or level-0 cells, sorted
  std::vector<i32> node_of_occ;   // occurrence (halo position * np + a, or cell * nn + b) -> node
  std::vector<i32> local;         // node -> local index (-1: not local or Dirichlet)
  i64 pos_of(i64 fam) const {
    auto it = std::lower_bound(halo.begin(), halo.end(), fam);
    GMG_REQUIRE(it != halo.end() && *it == fam, GMG_E_STATE, "family outside the halo");
    return (i64)(it - halo.begin());
  }
};

}  // namespace

void eig_start_from_keys(LocalTopo& T) {
  // R10b: -5.5 + (Morton key of the node on the level-l lattice mod 12) on owned S DoFs
  for (int l = 0; l <= T.L; ++l) {
    LocalLevel& v = T.lv[l];
    if (!v.eig_v.empty()) continue;
    v.eig_v.assign(v.n_local(), 0.0);
    for (i64 i = 0; i < v.n_owned; ++i) {
      if (v.cls[i] != CLS_S) continue;
      const Vec3 X = unmorton(T.dim, v.owned_key[i]);
      Vec3 Y{0, 0, 0};
      for (int j = 0; j < T.dim; ++j) Y[j] = X[j] >> (T.L - l);
      v.eig_v[i] = -5.5 + (double)(morton(T.dim, Y) % 12);
    }
  }
}

LocalTopo make_local_direct(const Forest& f, const Partition& p, int k, int rank, bool eig_key,
                            LocalCounts* counts) {
  GMG_REQUIRE(k == 1 || k == 2, GMG_E_INVALID_ARG, "k must be 1 or 2");
  const int d = f.dim, L = f.L, P = p.n_ranks;
  GMG_REQUIRE(rank >= 0 && rank < P, GMG_E_INVALID_ARG, "rank out of range");
  GMG_REQUIRE(eig_key, GMG_E_INVALID_ARG, "rank-local setup needs the key-based eigen start vector (R10b)");
  const i64 emax = std::max({f.ext[0], f.ext[1], f.ext[2]});
  const int cbits = bits_for((u64)(k * emax) << L);
  GMG_REQUIRE(cbits * d <= 64 && (d == 2 || cbits <= 21), GMG_E_DEPTH, "lattice keys exceed 64 bits");
  const int kbits = cbits * d;
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

  // ---------------- helpers over the global partition (cells of every level, SFC order;
  // the cells of level l >= 1 are families of nch consecutive children)
  auto nfam_of = [&](int l) -> i64 { return l == 0 ? 0 : (i64)p.levels[l].key.size() / nch; };
  auto comp = [&](int l, i64 fi) -> int { return p.levels[l].owner[(size_t)fi * nch]; };   // computing rank
  auto cell_index = [&](int l, u64 key) -> i64 {
    const auto& ks = p.levels[l].key;
    auto it = std::lower_bound(ks.begin(), ks.end(), key);
    return (it != ks.end() && *it == key) ? (i64)(it - ks.begin()) : -1;
  };
  auto parent_key = [&](int l, i64 fi) -> u64 { return p.levels[l].key[(size_t)fi * nch] >> d; };
  auto X_of = [&](const Vec3& G, int l, const std::array<int, 3>& off, int mult) {
    Vec3 X{0, 0, 0};
    for (int j = 0; j < d; ++j) X[j] = ((i64)mult * k * G[j] + off[j]) << (L - l);
    return X;
  };
  // level-0 local node b of a cell: offsets on the level-0 node lattice
  std::vector<std::array<int, 3>> off0(nn);
  for (int b = 0; b < nn; ++b) {
    int r = b;
    for (int j = 0; j < 3; ++j) {
      off0[b][j] = j < d ? r % (k + 1) : 0;
      if (j < d) r /= (k + 1);
    }
  }

  // ---------------- families computed here, per level (level 0: cells)
  std::vector<std::vector<i64>> mine(L + 1);
  for (i64 c = 0; c < (i64)p.levels[0].key.size(); ++c)
    if (p.levels[0].owner[c] == rank) mine[0].push_back(c);
  for (int l = 1; l <= L; ++l)
    for (i64 fi = 0; fi < nfam_of(l); ++fi)
      if (comp(l, fi) == rank) mine[l].push_back(fi);

  LevelKeep prev;   // level l-1
  std::vector<std::vector<i32>> leaf_run(L + 1);   // owned free leaf DoFs per level (local index)
  for (int l = 0; l <= L; ++l) {
    LocalLevel& v = Lt.lv[l];
    v.level = l;
    v.first_owned = -1;
    LevelKeep cur;
    const int stride = l == 0 ? nn : np;       // occurrences per halo entry
    // ---------------- halo and what this rank needs of it
    // needmask[h]: children of halo family h whose nodes this rank needs (parents of
    // its level-(l+1) families); ismine[h]: h computed here (its whole patch needed)
    std::vector<i64>& H = cur.halo;
    if (l == 0) {
      H.resize(p.levels[0].key.size());
      std::iota(H.begin(), H.end(), 0);
    } else {
      std::vector<i64> needfam = mine[l];
      if (l < L)
        for (i64 f1 : mine[l + 1]) needfam.push_back(cell_index(l, parent_key(l + 1, f1)) / nch);
      std::sort(needfam.begin(), needfam.end());
      needfam.erase(std::unique(needfam.begin(), needfam.end()), needfam.end());
      for (i64 fi : needfam) {
        const Vec3 G = unmorton(d, parent_key(l, fi));
        for (int o = 0; o < pt.ndir; ++o) {
          const Vec3 Q{G[0] + o % 3 - 1, G[1] + (o / 3) % 3 - 1, d == 3 ? G[2] + o / 9 - 1 : 0};
          if (!f.in_domain(l - 1, Q)) continue;
          const i64 c = cell_index(l, morton(d, Q) << d);
          if (c >= 0) H.push_back(c / nch);
        }
      }
      std::sort(H.begin(), H.end());
      H.erase(std::unique(H.begin(), H.end()), H.end());
    }
    const i64 nh = (i64)H.size();
    std::vector<uint8_t> ismine(nh, 0);
    std::vector<u32> needmask(nh, 0);
    if (l == 0) {
      for (i64 c : mine[0]) ismine[c] = 1;
      if (L >= 1)
        for (i64 f1 : mine[1]) ismine[cell_index(0, parent_key(1, f1))] = 1;   // a level-0 cell: all its nodes
    } else {
      for (i64 fi : mine[l]) ismine[cur.pos_of(fi)] = 1;
      if (l < L)
        for (i64 f1 : mine[l + 1]) {
          const i64 c = cell_index(l, parent_key(l + 1, f1));
          needmask[cur.pos_of(c / nch)] |= 1u << (c % nch);
        }
    }
    // per halo entry: computing rank, class masks, next-level computing rank per child
    std::vector<i32> hcomp(nh);
    std::vector<u32> hout(nh, 0), hleafn(nh, 0);
    std::vector<std::array<i32, 8>> hnext(nh);
    for (i64 h = 0; h < nh; ++h) {
      const i64 fi = H[h];
      hnext[h].fill(-1);
      if (l == 0) {
        hcomp[h] = 0;   // coarse handoff: level-0 DoFs owned by rank 0 (R25)
        continue;
      }
      hcomp[h] = comp(l, fi);
      const Vec3 G = unmorton(d, parent_key(l, fi));
      for (int o = 0; o < pt.ndir; ++o) {
        const Vec3 Q{G[0] + o % 3 - 1, G[1] + (o / 3) % 3 - 1, d == 3 ? G[2] + o / 9 - 1 : 0};
        if (Q == G) continue;
        if (!f.in_domain(l - 1, Q)) hout[h] |= 1u << o;
        else if (!f.is_refined(l - 1, morton(d, Q))) hleafn[h] |= 1u << o;
      }
      if (l < L)
        for (int c = 0; c < nch; ++c) {
          const size_t ci = (size_t)fi * nch + c;
          if (p.levels[l].leaf[ci]) continue;
          const i64 c1 = cell_index(l + 1, p.levels[l].key[ci] << d);
          if (c1 >= 0) hnext[h][c] = comp(l + 1, c1 / nch);
        }
    }
    // ---------------- occurrences, sorted by key -- in key-range chunks of at most
    // ~64M occurrences so that the sort buffers stay bounded (the finest level of a
    // config-5 rank has ~270M occurrences); every key falls into exactly one chunk,
    // so the nodes come out in key order across chunks
    const i64 n_occ = nh * stride;
    GMG_REQUIRE(n_occ < ((i64)1 << 32), GMG_E_OOM, "halo too large for 32-bit occurrence ids");
    auto occ_key = [&](i64 h, int a) {
      const Vec3 G = unmorton(d, l == 0 ? p.levels[0].key[H[h]] : parent_key(l, H[h]));
      const Vec3 X = l == 0 ? X_of(G, 0, off0[a], 1) : X_of(G, l, pt.pa[a], 2);
      return morton(d, X);
    };
    u64 kmin = ~0ull, kmax = 0;
    for (i64 h = 0; h < nh; ++h)
      for (int a = 0; a < stride; ++a) {
        const u64 kk = occ_key(h, a);
        kmin = std::min(kmin, kk);
        kmax = std::max(kmax, kk);
      }
    i64 chunk_target = (i64)1 << 26;
    if (const char* e = std::getenv("GMG_OCC_CHUNK")) chunk_target = std::max<i64>(64, std::atoll(e));   // tests
    const i64 n_chunks = n_occ == 0 ? 1 : std::max<i64>(1, (n_occ + chunk_target - 1) / chunk_target);
    const u64 span = n_occ == 0 ? 1 : (kmax - kmin) / (u64)n_chunks + 1;
    cur.node_of_occ.assign(n_occ, -1);
    std::vector<u64> nkey;
    std::vector<uint8_t> nfl, nneed, nmine;
    std::vector<i32> nown, ntpos;      // owner; transfer-owner family as halo position
    std::vector<std::vector<i32>> sidx(P);   // filled after local numbering: (node, peer)
    std::vector<std::pair<i32, i32>> sends;   // (peer, node) for owned nodes
    for (i64 ch = 0; ch < n_chunks; ++ch) {
    const u64 lo = kmin + span * (u64)ch, hi = ch + 1 == n_chunks ? ~0ull : kmin + span * (u64)(ch + 1);
    std::vector<u64> okey;
    std::vector<u32> oid;
    for (i64 h = 0; h < nh; ++h)
      for (int a = 0; a < stride; ++a) {
        const u64 kk = occ_key(h, a);
        if (kk < lo || kk >= hi) continue;
        okey.push_back(kk);
        oid.push_back((u32)(h * stride + a));
      }
    radix_sort_pairs32(okey, oid, kbits);
    const i64 n_run = (i64)okey.size();
    for (i64 s = 0; s < n_run;) {
      i64 e = s;
      while (e < n_run && okey[e] == okey[s]) ++e;
      uint8_t fl = 0, need = 0, inmine = 0;
      i32 own = INT32_MAX;
      const i32 node = (i32)nkey.size();
      for (i64 q = s; q < e; ++q) {
        const i64 h = oid[q] / stride;
        const int a = (int)(oid[q] % stride);
        cur.node_of_occ[oid[q]] = node;
        own = std::min(own, hcomp[h]);
        if (l == 0) {
          if (p.levels[0].leaf[H[h]]) fl |= F_LEAF;
        } else {
          if (pt.dirmask[a] & hout[h]) fl |= F_B;
          if (pt.dirmask[a] & hleafn[h]) fl |= F_EREG;
          for (int c = 0; c < nch; ++c)
            if ((pt.childmask[a] & (1u << c)) && p.levels[l].leaf[(size_t)H[h] * nch + c]) fl |= F_LEAF;
        }
        const bool m = ismine[h] != 0;
        const bool nc = l > 0 && (pt.childmask[a] & needmask[h]) != 0;
        if (m || nc) need = 1;
        if (m && hcomp[h] == rank) inmine = 1;
      }
      if (l == 0) {
        fl |= on_boundary(f, k, unmorton(d, okey[s])) ? F_B : 0;
        own = 0;
        inmine = rank == 0;
      }
      i32 tpos = INT32_MAX;
      if (l > 0)
        for (i64 q = s; q < e; ++q) {
          const i32 h = (i32)(oid[q] / stride);
          if (hcomp[h] == own) tpos = std::min(tpos, h);
        }
      // ranks needing an owned node: computing ranks of the containing families and
      // of the next-finer families of containing refined cells
      if (l > 0 && own == rank && inmine && !(fl & F_B)) {
        i32 qs[64];
        int nq = 0;
        for (i64 q = s; q < e; ++q) {
          const i64 h = oid[q] / stride;
          const int a = (int)(oid[q] % stride);
          if (hcomp[h] != rank && nq < 64) qs[nq++] = hcomp[h];
          for (int c = 0; c < nch; ++c)
            if ((pt.childmask[a] & (1u << c)) && hnext[h][c] >= 0 && hnext[h][c] != rank && nq < 64)
              qs[nq++] = hnext[h][c];
        }
        GMG_REQUIRE(nq < 64, GMG_E_STATE, "too many ranks share one node");
        if (nq) {
          std::sort(qs, qs + nq);
          nq = (int)(std::unique(qs, qs + nq) - qs);
          for (int t = 0; t < nq; ++t) sends.push_back({qs[t], node});
        }
      }
      nkey.push_back(okey[s]);
      nfl.push_back(fl);
      nown.push_back(own);
      ntpos.push_back(tpos);
      nneed.push_back(need);
      nmine.push_back(inmine);
      s = e;
    }
    }   // chunk
    const i64 nnodes = (i64)nkey.size();
    // ---------------- counts: each node by its owner (B nodes by the min computing rank)
    {
      const i64 cstep = (i64)1 << (L - l + 1);
      for (i64 i = 0; i < nnodes; ++i) {
        if (nown[i] != rank || !nmine[i]) continue;
        const uint8_t fl = nfl[i];
        const bool B = fl & F_B, E = fl & F_EREG, inleaf = fl & F_LEAF;
        if (B) cnt.B[l]++;
        else if (E) cnt.E[l]++;
        else cnt.S[l]++;
        if (!inleaf) continue;
        bool coarse = false;
        if (l > 0 && E) {
          const Vec3 X = unmorton(d, nkey[i]);
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
    std::vector<i64> owned, ghosts;
    for (i64 i = 0; i < nnodes; ++i) {
      if (nfl[i] & F_B) continue;
      if (nown[i] == rank && (l > 0 ? (nneed[i] && nmine[i]) : rank == 0)) owned.push_back(i);
      else if (nneed[i] && nown[i] != rank) ghosts.push_back(i);
    }
    std::stable_sort(ghosts.begin(), ghosts.end(), [&](i64 a, i64 b) { return nown[a] < nown[b]; });
    v.n_owned = (i64)owned.size();
    v.n_ghost = (i64)ghosts.size();
    const i64 nloc = v.n_local();
    cur.local.assign(nnodes, -1);
    for (i64 i = 0; i < v.n_owned; ++i) cur.local[owned[i]] = (i32)i;
    for (i64 i = 0; i < v.n_ghost; ++i) cur.local[ghosts[i]] = (i32)(v.n_owned + i);
    v.owned_key.resize(v.n_owned);
    v.ghost_key.resize(v.n_ghost);
    v.ghost_owner.resize(v.n_ghost);
    for (i64 i = 0; i < v.n_owned; ++i) v.owned_key[i] = nkey[owned[i]];
    for (i64 i = 0; i < v.n_ghost; ++i) {
      v.ghost_key[i] = nkey[ghosts[i]];
      v.ghost_owner[i] = nown[ghosts[i]];
    }
    // ---------------- exchange plan
    if (l == 0) {
      if (rank == 0)
        for (int q = 1; q < P; ++q) {
          // rank q needs the nodes of its level-0 cells and of the parents of its level-1 families
          std::vector<char> needc(nh, 0);
          for (i64 c = 0; c < nh; ++c)
            if (p.levels[0].owner[c] == q) needc[c] = 1;
          if (L >= 1)
            for (i64 fi = 0; fi < nfam_of(1); ++fi)
              if (comp(1, fi) == q) needc[cell_index(0, parent_key(1, fi))] = 1;
          std::vector<i32> ns;
          for (i64 c = 0; c < nh; ++c)
            if (needc[c])
              for (int b = 0; b < nn; ++b) ns.push_back(cur.node_of_occ[c * nn + b]);
          std::sort(ns.begin(), ns.end());
          ns.erase(std::unique(ns.begin(), ns.end()), ns.end());
          for (i32 i : ns)
            if (!(nfl[i] & F_B)) sidx[q].push_back(cur.local[i]);
        }
    } else {
      std::sort(sends.begin(), sends.end());   // by peer, then node (= key order)
      for (auto& pr : sends) sidx[pr.first].push_back(cur.local[pr.second]);
    }
    std::vector<i64> rcount(P, 0);
    for (i64 i = 0; i < v.n_ghost; ++i) rcount[v.ghost_owner[i]]++;
    v.send_off.push_back(0);
    v.recv_off.push_back(0);
    i64 gpos = 0;
    for (int q = 0; q < P; ++q) {
      if (rcount[q] == 0 && sidx[q].empty()) continue;
      v.peers.push_back(q);
      for (i32 s2 : sidx[q]) v.send_idx.push_back(s2);
      for (i64 c = 0; c < rcount[q]; ++c) v.recv_idx.push_back((i32)(v.n_owned + gpos + c));
      gpos += rcount[q];
      v.send_off.push_back((i64)v.send_idx.size());
      v.recv_off.push_back((i64)v.recv_idx.size());
    }
    // ---------------- local cells, classes, lambda, eigen start vector
    v.cls.resize(nloc);
    v.lam.assign(nloc, 0);
    // eig_v stays empty: the key-based start vector (R10b) is formed from owned_key
    // where it is needed (eig_start_from_keys), not stored for all local DoFs
    auto fill_node = [&](i64 li, i64 i) {
      const uint8_t fl = nfl[i];
      v.cls[li] = (fl & F_EREG) ? CLS_E : CLS_S;
      if (li >= v.n_owned || v.cls[li] != CLS_S) return;
      v.lam[li] = (fl & F_LEAF) ? 1 : 0;   // S here, in a level-l leaf: not S on level l+1
    };
    for (i64 i = 0; i < v.n_owned; ++i) fill_node(i, owned[i]);
    for (i64 i = 0; i < v.n_ghost; ++i) fill_node(v.n_owned + i, ghosts[i]);
    for (i64 i = 0; i < v.n_owned; ++i)
      if (v.cls[i] == CLS_S) cnt.own_S[l]++;
    if (l == 0) {
      for (i64 c : mine[0]) v.cell_global.push_back(c);
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
        const i64 occ = l == 0 ? gc * nn + b : cur.pos_of(gc / nch) * np + pt.cell_to_patch[gc % nch][b];
        const i32 i = cur.node_of_occ[occ];
        v.cell_dofs[(size_t)c * nn + b] = (nfl[i] & F_B) ? -1 : cur.local[i];
      }
      if (p.levels[l].leaf[gc]) v.leaf_cells.push_back((i32)c);
    }
    if (l > 0) {
      const int row = np + nn;
      v.xfer.resize((size_t)v.n_fam * row);
      for (i64 lf = 0; lf < v.n_fam; ++lf) {
        const i64 fi = mine[l][lf];
        const i64 hp = cur.pos_of(fi);
        bool edge = false;
        for (int a = 0; a < np; ++a) {
          const i32 i = cur.node_of_occ[hp * np + a];
          i32 enc = -1;
          if (!(nfl[i] & F_B)) {
            const i32 lg = cur.local[i];
            GMG_REQUIRE(lg >= 0, GMG_E_STATE, "patch node without a local index");
            const bool towner = ntpos[i] == (i32)hp;
            enc = towner ? lg : -2 - lg;
            if (towner) {
              GMG_REQUIRE(lg < v.n_owned, GMG_E_STATE, "transfer owner is not the DoF owner");
              if (nfl[i] & F_EREG) edge = true;
            }
          }
          v.xfer[(size_t)lf * row + a] = enc;
        }
        // the parent's (k+1)^d nodes on level l-1
        const i64 pc = cell_index(l - 1, parent_key(l, fi));
        for (int b = 0; b < nn; ++b) {
          const i64 occ = l - 1 == 0 ? pc * nn + b : prev.pos_of(pc / nch) * np + pt.cell_to_patch[pc % nch][b];
          const i32 i = prev.node_of_occ[occ];
          v.xfer[(size_t)lf * row + np + b] = prev.local[i];
        }
        if (edge) v.edge_fams.push_back((i32)lf);
      }
      // complete grandfamilies (as make_local)
      if (d == 3 && l >= 2)
        for (i64 lf = 0; lf + 7 < v.n_fam;) {
          const u64 k0 = parent_key(l, mine[l][lf]);
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
    // ---------------- owned free leaf DoFs of this level
    for (i64 i = 0; i < v.n_owned; ++i)
      if (v.lam[i]) leaf_run[l].push_back((i32)i);   // owned order = key order
    cnt.own_dofs[l] = (double)v.n_owned;
    // the Dirichlet nodes have local -1: prev.local gives -1 for them (xfer parent part)
    for (i64 i = 0; i < nnodes; ++i)
      if (nfl[i] & F_B) cur.local[i] = -1;
    prev = std::move(cur);
  }
  // leaf order (owner, key): merge the per-level runs (each in key order) by key
  {
    size_t total = 0;
    for (auto& r : leaf_run) total += r.size();
    Lt.leaf_level.reserve(total);
    Lt.leaf_local.reserve(total);
    Lt.leaf_key.reserve(total);
    std::vector<size_t> pos(L + 1, 0);
    for (size_t c = 0; c < total; ++c) {
      int best = -1;
      u64 bk = ~0ull;
      for (int l = 0; l <= L; ++l)
        if (pos[l] < leaf_run[l].size()) {
          const u64 kk = Lt.lv[l].owned_key[leaf_run[l][pos[l]]];
          if (best < 0 || kk < bk) {
            best = l;
            bk = kk;
          }
        }
      Lt.leaf_level.push_back((int8_t)best);
      Lt.leaf_local.push_back(leaf_run[best][pos[best]]);
      Lt.leaf_key.push_back(bk);
      ++pos[best];
    }
  }
  Lt.n_leaf_owned = (i64)Lt.leaf_level.size();
  Lt.leaf_first = -1;          // set from the other ranks' counts (LocalCounts)
  Lt.n_leaf_global = -1;
  cnt.leaf_free = (double)Lt.n_leaf_owned;
  if (counts) *counts = cnt;
  return Lt;
}

}  // namespace gmg
