// SFC partition with the first-child rule and the partition-efficiency model.
//
// leaves distributed along the space-filling curve; every parent is
// owned by the owner of its first child, recursively.  Here computed directly
// as "owner of the first SFC leaf of the subtree" (the first leaf of a cell's
// subtree starts at the cell's lower corner in padded Morton order).
// N_l, N_{l,p}, W_opt, W_sync, W_l, W, eta (exact integers).
#include <numeric>

#include "forest.hpp"

namespace gmg {

Partition make_partition(const Forest& f, int n_ranks, int mode, i64 coarse_cells) {
  GMG_REQUIRE(n_ranks >= 1, GMG_E_INVALID_ARG, "n_ranks must be >= 1");
  GMG_REQUIRE(mode == GMG_PARTITION_FIRST_CHILD || mode == GMG_PARTITION_PER_LEVEL, GMG_E_INVALID_ARG,
              "partition mode");
  Partition p;
  p.f = &f;
  p.n_ranks = n_ranks;
  p.mode = mode;
  const i64 N = f.n_leaves();
  p.leaf_owner.resize(N);
  {
    i64 base = N / n_ranks, rem = N % n_ranks, pos = 0;
    for (int r = 0; r < n_ranks; ++r) {
      i64 cnt = base + (r < rem ? 1 : 0);
      for (i64 i = 0; i < cnt; ++i) p.leaf_owner[pos++] = r;
    }
  }
  const int d = f.dim, L = f.L;
  // padded leaf keys (sorted)
  std::vector<u64> lk(N);
  for (i64 i = 0; i < N; ++i) {
    Vec3 g = f.gc[i];
    lk[i] = morton(d, g) << (d * (L - f.level[i]));
  }
  p.levels.resize(L + 1);
  for (int l = 0; l <= L; ++l) {
    auto& lc = p.levels[l];
    // merge refined cells and leaves of level l (both sorted)
    std::vector<u64> leafk;
    for (i64 i = 0; i < N; ++i)
      if (f.level[i] == l) leafk.push_back(morton(d, f.gc[i]));
    // leaves are in SFC order; cells of one level in SFC order are Morton-sorted
    const auto& rk = f.refined[l];
    lc.key.resize(leafk.size() + rk.size());
    lc.leaf.resize(lc.key.size());
    size_t a = 0, b = 0, o = 0;
    while (a < leafk.size() || b < rk.size()) {
      if (b >= rk.size() || (a < leafk.size() && leafk[a] < rk[b])) {
        lc.key[o] = leafk[a++];
        lc.leaf[o++] = 1;
      } else {
        lc.key[o] = rk[b++];
        lc.leaf[o++] = 0;
      }
    }
    lc.owner.resize(lc.key.size());
    for (size_t c = 0; c < lc.key.size(); ++c) {
      u64 pk = lc.key[c] << (d * (L - l));
      auto it = std::lower_bound(lk.begin(), lk.end(), pk);
      GMG_REQUIRE(it != lk.end() && *it == pk, GMG_E_STATE, "first leaf of subtree not found");
      lc.owner[c] = p.leaf_owner[it - lk.begin()];
    }
    if (mode == GMG_PARTITION_PER_LEVEL) {
      // P:597 alternative (reading R29): every level partitioned on its own along the
      // SFC, whole families (children of one parent; single cells on level 0) kept
      // together: the family starting at cell index c (of N_l) goes to rank
      // floor(n_ranks * c / N_l).
      const i64 n = (i64)lc.key.size();
      for (i64 c = 0; c < n;) {
        i64 e = c + 1;
        if (l > 0)
          while (e < n && (lc.key[e] >> d) == (lc.key[c] >> d)) ++e;
        const i32 r = (i32)((__int128)n_ranks * c / n);
        for (i64 q = c; q < e; ++q) lc.owner[q] = r;
        c = e;
      }
    }
  }
  // coarse-level gather ("processors drop out automatically on coarser levels",
  // P:616-617, taken to its end): the levels from 0 up to the last one with at most
  // coarse_cells cells live entirely on rank 0, so the small levels of the V-cycle
  // run without exchanges; the handoff to the finer levels is the ordinary
  // restriction / prolongation ghost exchange of the first finer level
  if (coarse_cells > 0)
    for (int l = 0; l <= L && (i64)p.levels[l].key.size() <= coarse_cells; ++l)
      std::fill(p.levels[l].owner.begin(), p.levels[l].owner.end(), 0);
  p.coarse_cells = coarse_cells;
  return p;
}

gmg_model partition_model(const Partition& p, i64 W0_override) {
  gmg_model m;
  std::memset(&m, 0, sizeof m);
  const int nl = (int)p.levels.size();
  GMG_REQUIRE(nl <= GMG_MAX_LEVELS, GMG_E_DEPTH, "too many levels");
  const int P = p.n_ranks;
  m.n_levels = nl;
  m.n_ranks = P;
  std::vector<i64> tally((size_t)nl * P, 0);
  for (int l = 0; l < nl; ++l) {
    for (i32 o : p.levels[l].owner) tally[(size_t)l * P + o]++;
    m.N[l] = (i64)p.levels[l].key.size();
    i64 w = 0;
    for (int r = 0; r < P; ++r) w = std::max(w, tally[(size_t)l * P + r]);
    m.W_l[l] = w;
  }
  i64 w0_opt, w0_sync, w0;
  if (W0_override < 0) {
    w0_opt = m.N[0];
    w0_sync = (m.N[0] + P - 1) / P;
    w0 = m.W_l[0];
  } else {
    w0_opt = w0_sync = w0 = W0_override;
  }
  i64 num = w0_opt, sync = w0_sync, W = w0;
  for (int l = 1; l < nl; ++l) {
    num += m.N[l];
    sync += (m.N[l] + P - 1) / P;
    W += m.W_l[l];
  }
  i64 g = std::gcd(num, (i64)P);
  m.W_opt_num = num / g;
  m.W_opt_den = P / g;
  m.W_sync = sync;
  m.W = W;
  // eta = num / (P W)
  i64 en = num, ed = (i64)P * W;
  i64 g2 = std::gcd(en, ed);
  m.eta_num = en / g2;
  m.eta_den = ed / g2;
  // ghost children
  const int d = p.f->dim;
  for (int l = 1; l < nl; ++l) {
    const auto& ch = p.levels[l];
    const auto& pa = p.levels[l - 1];
    i64 gh = 0;
    size_t pi = 0;
    for (size_t c = 0; c < ch.key.size(); ++c) {
      u64 pk = ch.key[c] >> d;
      while (pi < pa.key.size() && pa.key[pi] < pk) ++pi;
      GMG_REQUIRE(pi < pa.key.size() && pa.key[pi] == pk, GMG_E_STATE, "parent not found");
      gh += ch.owner[c] != pa.owner[pi];
    }
    m.ghost_children[l] = gh;
    m.children[l] = (i64)ch.key.size();
  }
  return m;
}

}  // namespace gmg
