// Forest construction, refinement recipes and 2:1 vertex-balance closure.
//
// Paper: refinement tree / forest and levels, isotropic 2^d
// refinement, closure to one-irregularity "if they share a degree
// of freedom" (read as vertex balance, R5), z-curve order
// (P:603).
//
// Balance is enforced through an equivalent condition on refined cells: a
// forest is 2:1 vertex balanced iff every refined cell P of level >= 1 has all
// 3^d - 1 same-level neighbours existing as cells (their parents refined).
// (A leaf T of level l touches a leaf of level <= l-2 exactly when some
// level-(l-1) cell adjacent to T's parent does not exist.)
#include <algorithm>
#include <numeric>

#include <functional>

#include "forest.hpp"

namespace gmg {

std::vector<u64> FlatSet::sorted_keys() const {
  std::vector<u64> out;
  out.reserve(count);
  for (u64 k : slot)
    if (k != EMPTY) out.push_back(k);
  std::sort(out.begin(), out.end());
  return out;
}

void radix_sort_pairs(std::vector<u64>& key, std::vector<u64>& val, int key_bits) {
  const size_t n = key.size();
  std::vector<u64> k2(n), v2(n);
  const int RB = 11, R = 1 << RB;
  std::vector<size_t> cnt(R);
  for (int shift = 0; shift < key_bits; shift += RB) {
    std::fill(cnt.begin(), cnt.end(), 0);
    for (size_t i = 0; i < n; ++i) cnt[(key[i] >> shift) & (R - 1)]++;
    size_t s = 0;
    for (int b = 0; b < R; ++b) { size_t c = cnt[b]; cnt[b] = s; s += c; }
    for (size_t i = 0; i < n; ++i) {
      size_t d = cnt[(key[i] >> shift) & (R - 1)]++;
      k2[d] = key[i];
      v2[d] = val[i];
    }
    key.swap(k2);
    val.swap(v2);
  }
}

void radix_sort_keys(std::vector<u64>& key, int key_bits) {
  const size_t n = key.size();
  std::vector<u64> k2(n);
  const int RB = 11, R = 1 << RB;
  std::vector<size_t> cnt(R);
  for (int shift = 0; shift < key_bits; shift += RB) {
    std::fill(cnt.begin(), cnt.end(), 0);
    for (size_t i = 0; i < n; ++i) cnt[(key[i] >> shift) & (R - 1)]++;
    size_t s = 0;
    for (int b = 0; b < R; ++b) { size_t c = cnt[b]; cnt[b] = s; s += c; }
    for (size_t i = 0; i < n; ++i) k2[cnt[(key[i] >> shift) & (R - 1)]++] = key[i];
    key.swap(k2);
  }
}

int Forest::tree_of(const Vec3& tpos) const {
  for (size_t t = 0; t < trees.size(); ++t)
    if (trees[t][0] == tpos[0] && trees[t][1] == tpos[1] && trees[t][2] == tpos[2]) return (int)t;
  return -1;
}

static Forest domain_of(int dim, const std::vector<Vec3>& trees_in) {
  Forest f;
  f.dim = dim;
  GMG_REQUIRE(dim == 2 || dim == 3, GMG_E_INVALID_ARG, "dim must be 2 or 3");
  GMG_REQUIRE(!trees_in.empty(), GMG_E_INVALID_ARG, "need at least one tree");
  std::vector<std::pair<u64, Vec3>> t;
  Vec3 ext{1, 1, 1};
  for (auto p : trees_in) {
    for (int j = 0; j < dim; ++j) {
      GMG_REQUIRE(p[j] >= 0 && p[j] < 8, GMG_E_INVALID_ARG, "tree coordinates must be in [0,8)");
      ext[j] = std::max<i64>(ext[j], p[j] + 1);
    }
    if (dim == 2) p[2] = 0;
    t.push_back({morton(dim, p), p});
  }
  std::sort(t.begin(), t.end(), [](auto& a, auto& b) { return a.first < b.first; });
  for (size_t i = 1; i < t.size(); ++i)
    GMG_REQUIRE(t[i].first != t[i - 1].first, GMG_E_INVALID_ARG, "duplicate tree position");
  for (auto& x : t) f.trees.push_back(x.second);
  f.ext = ext;
  f.occ.assign((size_t)(ext[0] * ext[1] * ext[2]), 0);
  for (auto& p : f.trees) f.occ[(size_t)((p[2] * ext[1] + p[1]) * ext[0] + p[0])] = 1;
  return f;
}

Forest forest_from_refined(int dim, const std::vector<Vec3>& trees, std::vector<FlatSet>& R) {
  Forest f = domain_of(dim, trees);
  // cells level by level; leaves = cells that are not refined
  std::vector<Vec3> cur(f.trees.begin(), f.trees.end());
  std::vector<int8_t> lev;
  std::vector<Vec3> gc;
  int l = 0;
  while (!cur.empty()) {
    std::vector<Vec3> next;
    for (auto& g : cur) {
      u64 key = morton(dim, g);
      if (l < (int)R.size() && R[l].contains(key)) {
        for (int c = 0; c < (1 << dim); ++c) {
          Vec3 h{2 * g[0] + (c & 1), 2 * g[1] + ((c >> 1) & 1), dim == 3 ? 2 * g[2] + ((c >> 2) & 1) : 0};
          next.push_back(h);
        }
      } else {
        lev.push_back((int8_t)l);
        gc.push_back(g);
      }
    }
    cur.swap(next);
    ++l;
  }
  f.L = 0;
  for (auto v : lev) f.L = std::max<int>(f.L, v);
  GMG_REQUIRE((dim == 3 && f.L <= 19) || (dim == 2 && f.L <= 29), GMG_E_DEPTH,
              "level too deep for 64-bit lattice keys");
  // SFC order: Morton of the lower corner on the finest lattice
  const size_t n = lev.size();
  std::vector<u64> key(n), idx(n);
  for (size_t i = 0; i < n; ++i) {
    Vec3 g = gc[i];
    for (int j = 0; j < dim; ++j) g[j] <<= (f.L - lev[i]);
    key[i] = morton(dim, g);
    idx[i] = i;
  }
  radix_sort_pairs(key, idx, bits_for((u64)std::max({f.ext[0], f.ext[1], f.ext[2]}) << f.L) * dim);
  f.level.resize(n);
  f.gc.resize(n);
  for (size_t i = 0; i < n; ++i) {
    f.level[i] = lev[idx[i]];
    f.gc[i] = gc[idx[i]];
  }
  f.refined.resize(f.L + 1);
  for (int m = 0; m <= f.L && m < (int)R.size(); ++m) f.refined[m] = R[m].sorted_keys();
  return f;
}

static void ensure_refined(int dim, std::vector<FlatSet>& R, std::vector<std::pair<int, u64>>& work,
                           int l, Vec3 g) {
  while (true) {
    if ((int)R.size() <= l) R.resize(l + 1);
    u64 key = morton(dim, g);
    if (!R[l].insert(key)) return;
    work.push_back({l, key});
    if (l == 0) return;
    // the cell exists only if its parent is refined
    for (int j = 0; j < dim; ++j) g[j] >>= 1;
    --l;
  }
}

i64 close_balance(int dim, const Forest& dom, std::vector<FlatSet>& R,
                  std::vector<std::pair<int, u64>>& work) {
  i64 added = 0;
  const int nd = dim == 2 ? 9 : 27;
  while (!work.empty()) {
    auto [l, key] = work.back();
    work.pop_back();
    if (l == 0) continue;   // level-0 neighbours are trees: they always exist
    Vec3 g = unmorton(dim, key);
    for (int o = 0; o < nd; ++o) {
      Vec3 off{o % 3 - 1, (o / 3) % 3 - 1, dim == 3 ? o / 9 - 1 : 0};
      if (off[0] == 0 && off[1] == 0 && off[2] == 0) continue;
      Vec3 q{g[0] + off[0], g[1] + off[1], g[2] + off[2]};
      if (!dom.in_domain(l, q)) continue;
      Vec3 pq{q[0] >> 1, q[1] >> 1, q[2] >> 1};
      size_t before = work.size();
      if ((int)R.size() <= l - 1) R.resize(l);
      if (!R[l - 1].contains(morton(dim, pq))) {
        ensure_refined(dim, R, work, l - 1, pq);
        added += (i64)(work.size() - before);
      }
    }
  }
  return added;
}

// ------------------------------------------------------------------ recipes
using i128 = __int128;

static bool pred_center_ball(const gmg_recipe& r, int dim, int l, const Vec3& g) {
  i64 D = 1;
  for (int j = 0; j < dim; ++j) D = std::lcm(D, r.center_den[j]);
  i128 two = (i128)1 << (l + 1);
  i128 sum = 0;
  for (int j = 0; j < dim; ++j) {
    i128 num = (i128)(2 * g[j] + 1) * D - (i128)r.center_num[j] * (D / r.center_den[j]) * two;
    sum += num * num;
  }
  i128 lhs = sum * ((i128)r.radius_den * r.radius_den);
  i128 rr = (i128)r.radius_num * r.radius_num;
  i128 sc = (i128)D * two;
  return lhs <= rr * sc * sc;
}

static bool pred_sphere_surface(const gmg_recipe& r, int dim, int l, const Vec3& g) {
  i64 D = 1;
  for (int j = 0; j < dim; ++j) D = std::lcm(D, r.center_den[j]);
  i128 twol = (i128)1 << l;
  i128 mn = 0, mx = 0;
  for (int j = 0; j < dim; ++j) {
    i128 c = (i128)r.center_num[j] * (D / r.center_den[j]) * twol;
    i128 lo = (i128)g[j] * D, hi = (i128)(g[j] + 1) * D;
    i128 a = lo - c, b = c - hi;
    i128 dmin = a > b ? a : b;
    if (dmin < 0) dmin = 0;
    mn += dmin * dmin;
    i128 aa = a * a, bb = b * b;
    mx += aa > bb ? aa : bb;
  }
  i128 den = (i128)r.radius_den * r.shell_den;
  i128 rhi = (i128)r.radius_num * r.shell_den + (i128)r.shell_num * r.radius_den;
  i128 rlo = (i128)r.radius_num * r.shell_den - (i128)r.shell_num * r.radius_den;
  i128 unit = (i128)D * twol;
  bool cmin = mn * den * den <= (rhi * unit) * (rhi * unit);
  bool cmax = rlo <= 0 ? true : (mx * den * den >= (rlo * unit) * (rlo * unit));
  return cmin && cmax;
}

static bool pred_corner_dist(const gmg_recipe& r, int dim, int l, const Vec3& g) {
  if (l >= r.lmax) return false;
  i128 d2 = 0;
  for (int j = 0; j < dim; ++j) {
    i128 c = (i128)r.corner[j] << l;
    i128 v = std::max<i128>(std::max<i128>((i128)g[j] - c, c - ((i128)g[j] + 1)), 0);
    d2 += v * v;
  }
  return d2 <= ((i128)1 << (2 * r.s));
}

Forest forest_generate(const gmg_recipe& r) {
  const int dim = r.dim;
  GMG_REQUIRE(dim == 2 || dim == 3, GMG_E_INVALID_ARG, "recipe dim");
  GMG_REQUIRE(r.n_trees >= 1 && r.n_trees <= 8, GMG_E_INVALID_ARG, "recipe n_trees");
  std::vector<Vec3> trees;
  for (int t = 0; t < r.n_trees; ++t)
    trees.push_back({r.tree_xyz[3 * t], r.tree_xyz[3 * t + 1], dim == 3 ? r.tree_xyz[3 * t + 2] : 0});
  Forest dom = domain_of(dim, trees);
  std::vector<FlatSet> R(1);
  std::vector<std::pair<int, u64>> work;
  // global refinements: refine every cell of levels 0..g-1
  {
    std::vector<Vec3> cur = dom.trees;
    for (int l = 0; l < r.global_refinements; ++l) {
      if ((int)R.size() <= l) R.resize(l + 1);
      std::vector<Vec3> next;
      for (auto& g : cur) {
        R[l].insert(morton(dim, g));
        for (int c = 0; c < (1 << dim); ++c)
          next.push_back({2 * g[0] + (c & 1), 2 * g[1] + ((c >> 1) & 1),
                          dim == 3 ? 2 * g[2] + ((c >> 2) & 1) : 0});
      }
      cur.swap(next);
    }
  }
  Forest f = forest_from_refined(dim, trees, R);
  int passes = 0;
  while (r.rule != GMG_RULE_NONE && (r.n_passes < 0 || passes < r.n_passes)) {
    bool any = false;
    for (i64 i = 0; i < f.n_leaves(); ++i) {
      int l = f.level[i];
      const Vec3& g = f.gc[i];
      bool m = false;
      switch (r.rule) {
        case GMG_RULE_CENTER_BALL: m = pred_center_ball(r, dim, l, g); break;
        case GMG_RULE_SPHERE_SURFACE: m = pred_sphere_surface(r, dim, l, g); break;
        case GMG_RULE_CORNER_DIST: m = pred_corner_dist(r, dim, l, g); break;
        default: fail(GMG_E_INVALID_ARG, "unknown rule");
      }
      if (m) {
        if ((int)R.size() <= l) R.resize(l + 1);
        if (R[l].insert(morton(dim, g))) work.push_back({l, morton(dim, g)});
        any = true;
      }
    }
    if (!any) break;
    close_balance(dim, dom, R, work);
    f = forest_from_refined(dim, trees, R);
    ++passes;
  }
  return f;
}

// ------------------------------------------------------------------ mesh sequences
// The refinement sequences of the paper's partitioning study, on one
// coarse cell read as [-1,1]^d (the "negative quadrant" and the annulus radii
// need the origin at the cell centre; reading R27).  A level-l cell with global
// coordinates G spans x in [(2G - 2^l), (2G + 2 - 2^l)] / 2^l per direction.
static void refine_marked(int dim, const Forest& dom, std::vector<FlatSet>& R, const Forest& f,
                          const std::function<bool(int, const Vec3&)>& mark) {
  std::vector<std::pair<int, u64>> work;
  for (i64 i = 0; i < f.n_leaves(); ++i) {
    const int l = f.level[i];
    if (!mark(l, f.gc[i])) continue;
    if ((int)R.size() <= l) R.resize(l + 1);
    const u64 key = morton(dim, f.gc[i]);
    if (R[l].insert(key)) work.push_back({l, key});
  }
  close_balance(dim, dom, R, work);
}

Forest forest_sequence(int dim, gmg_sequence kind, int L) {
  GMG_REQUIRE(dim == 2 || dim == 3, GMG_E_INVALID_ARG, "sequence dim");
  GMG_REQUIRE(L >= 1 && L <= (dim == 3 ? 19 : 29), GMG_E_INVALID_ARG, "sequence level");
  GMG_REQUIRE(kind != GMG_SEQ_ANNULUS || L >= 4, GMG_E_INVALID_ARG, "annulus needs L >= 4");
  const std::vector<Vec3> trees{{0, 0, 0}};
  Forest dom = domain_of(dim, trees);
  std::vector<FlatSet> R(1);
  Forest f = forest_from_refined(dim, trees, R);
  auto step = [&](const std::function<bool(int, const Vec3&)>& mark) {
    refine_marked(dim, dom, R, f, mark);
    f = forest_from_refined(dim, trees, R);
  };
  auto all = [](int, const Vec3&) { return true; };
  // |centre|^2 * 4^l  (integer): centre x_j = (2 G_j + 1 - 2^l) / 2^l
  auto centre2 = [dim](int l, const Vec3& g) {
    i128 s = 0;
    for (int j = 0; j < dim; ++j) {
      const i128 n = 2 * (i128)g[j] + 1 - ((i128)1 << l);
      s += n * n;
    }
    return s;
  };
  auto centre_in = [&](int l, const Vec3& g, i128 num, i128 den) {   // |c|^2 <= num/den
    return centre2(l, g) * den <= num * ((i128)1 << (2 * l));
  };
  auto centre_out = [&](int l, const Vec3& g, i128 num, i128 den) {  // |c|^2 >= num/den
    return centre2(l, g) * den >= num * ((i128)1 << (2 * l));
  };
  switch (kind) {
    case GMG_SEQ_UNIFORM:                       // "global refinement of the coarse mesh L times"
      for (int i = 0; i < L; ++i) step(all);
      break;
    case GMG_SEQ_CIRCLE: {                      // "all mesh cells with at least one point inside the
      const long double rho2 = 1.0L / (16.0L * 3.14159265358979323846264338327950288L *
                                       3.14159265358979323846264338327950288L);   // (1/(4 pi))^2
      for (int i = 0; i < L; ++i)               //  circle of radius 1/(4 pi) around the origin"
        step([&](int l, const Vec3& g) {
          i128 d2 = 0;                          // (distance of the closed box to 0)^2 * 4^l
          for (int j = 0; j < dim; ++j) {
            const i128 lo = 2 * (i128)g[j] - ((i128)1 << l), hi = lo + 2;
            const i128 v = lo > 0 ? lo : (hi < 0 ? -hi : 0);
            d2 += v * v;
          }
          return (long double)d2 < rho2 * (long double)((i128)1 << (2 * l));   // irrational: no ties
        });
      break;
    }
    case GMG_SEQ_QUADRANT:                      // "after one uniform refinement ... refine the cell in
      step(all);                                //  the negative quadrant L-1 times"
      for (int i = 1; i < L; ++i)
        step([&](int l, const Vec3& g) {
          for (int j = 0; j < dim; ++j)
            if (2 * (i128)g[j] + 2 - ((i128)1 << l) > 0) return false;   // box inside [-1,0]^d
          return true;
        });
      break;
    case GMG_SEQ_ANNULUS:                       // L-3 uniform refinements, then three centre rules
      for (int i = 0; i < L - 3; ++i) step(all);
      step([&](int l, const Vec3& g) { return centre_in(l, g, 121, 400); });               // r <= 0.55
      step([&](int l, const Vec3& g) {
        return centre_out(l, g, 9, 100) && centre_in(l, g, 1849, 10000);                  // 0.3 .. 0.43
      });
      step([&](int l, const Vec3& g) {
        return centre_out(l, g, 4489, 40000) && centre_in(l, g, 1521, 10000);             // 0.335 .. 0.39
      });
      break;
    default:
      fail(GMG_E_INVALID_ARG, "unknown sequence");
  }
  return f;
}

Forest forest_create(int dim, int n_trees, const int32_t* tree_xyz, i64 n_leaves,
                     const int32_t* leaf_tree, const int8_t* leaf_level, const uint64_t* leaf_morton,
                     uint32_t flags) {
  GMG_REQUIRE(dim == 2 || dim == 3, GMG_E_INVALID_ARG, "dim must be 2 or 3");
  GMG_REQUIRE(n_trees >= 1 && tree_xyz, GMG_E_INVALID_ARG, "trees");
  GMG_REQUIRE(n_leaves >= 1 && leaf_tree && leaf_level && leaf_morton, GMG_E_INVALID_ARG, "leaves");
  std::vector<Vec3> trees;
  for (int t = 0; t < n_trees; ++t)
    trees.push_back({tree_xyz[dim * t], tree_xyz[dim * t + 1], dim == 3 ? tree_xyz[dim * t + 2] : 0});
  Forest dom = domain_of(dim, trees);
  const int maxL = dim == 3 ? 19 : 29;
  int L = 0;
  for (i64 i = 0; i < n_leaves; ++i) {
    GMG_REQUIRE(leaf_tree[i] >= 0 && leaf_tree[i] < n_trees, GMG_E_INVALID_ARG, "leaf_tree out of range");
    GMG_REQUIRE(leaf_level[i] >= 0, GMG_E_INVALID_ARG, "negative level");
    GMG_REQUIRE(leaf_level[i] <= maxL, GMG_E_DEPTH, "level too deep for 64-bit lattice keys");
    GMG_REQUIRE(leaf_morton[i] < (1ull << (dim * leaf_level[i])) || leaf_level[i] == 0,
                GMG_E_INVALID_ARG, "morton code out of range for its level");
    GMG_REQUIRE(leaf_level[i] > 0 || leaf_morton[i] == 0, GMG_E_INVALID_ARG, "morton of a root");
    L = std::max<int>(L, leaf_level[i]);
  }
  // sortedness first: (tree, padded Morton key) strictly increasing
  for (i64 i = 1; i < n_leaves; ++i) {
    GMG_REQUIRE(leaf_tree[i] >= leaf_tree[i - 1], GMG_E_UNSORTED, "leaves not sorted by tree");
    if (leaf_tree[i] == leaf_tree[i - 1]) {
      u64 a = leaf_morton[i - 1] << (dim * (L - leaf_level[i - 1]));
      u64 b = leaf_morton[i] << (dim * (L - leaf_level[i]));
      GMG_REQUIRE(b > a, GMG_E_UNSORTED, "leaves not strictly increasing in SFC order");
    }
  }
  // global coordinates and tiling per tree
  std::vector<Vec3> gc(n_leaves);
  u64 prev_key = 0;
  i64 prev_tree = -1;
  u64 expect = 0;
  for (i64 i = 0; i < n_leaves; ++i) {
    int l = leaf_level[i];
    Vec3 loc = unmorton(dim, leaf_morton[i]);
    const Vec3& tp = dom.trees[leaf_tree[i]];
    Vec3 g{(tp[0] << l) + loc[0], (tp[1] << l) + loc[1], dim == 3 ? (tp[2] << l) + loc[2] : 0};
    gc[i] = g;
    Vec3 s = g;
    for (int j = 0; j < dim; ++j) s[j] <<= (L - l);
    u64 key = morton(dim, s);
    u64 span = 1ull << (dim * (L - l));
    if (leaf_tree[i] != prev_tree) {
      GMG_REQUIRE(leaf_tree[i] > prev_tree, GMG_E_UNSORTED, "leaves not sorted by tree");
      if (prev_tree >= 0) {
        Vec3 te = dom.trees[prev_tree];
        Vec3 ts{te[0] << L, te[1] << L, te[2] << L};
        GMG_REQUIRE(expect == morton(dim, ts) + (1ull << (dim * L)), GMG_E_NOT_TILING,
                    "tree not completely covered by its leaves");
      }
      GMG_REQUIRE(leaf_tree[i] == prev_tree + 1, GMG_E_NOT_TILING, "tree without leaves");
      Vec3 ts{tp[0] << L, tp[1] << L, tp[2] << L};
      expect = morton(dim, ts);
      prev_tree = leaf_tree[i];
    } else {
      GMG_REQUIRE(key > prev_key, GMG_E_UNSORTED, "leaves not strictly increasing in SFC order");
    }
    GMG_REQUIRE(key == expect, key < expect ? GMG_E_NOT_TILING : GMG_E_NOT_TILING,
                "leaves overlap or leave a hole");
    expect = key + span;
    prev_key = key;
  }
  {
    GMG_REQUIRE(prev_tree == n_trees - 1, GMG_E_NOT_TILING, "trees without leaves");
    Vec3 te = dom.trees[prev_tree];
    Vec3 ts{te[0] << L, te[1] << L, te[2] << L};
    GMG_REQUIRE(expect == morton(dim, ts) + (1ull << (dim * L)), GMG_E_NOT_TILING,
                "tree not completely covered by its leaves");
  }
  // refined cells = proper ancestors of the leaves
  std::vector<FlatSet> R(L + 1);
  std::vector<std::pair<int, u64>> work;
  for (i64 i = 0; i < n_leaves; ++i) {
    Vec3 g = gc[i];
    for (int l = leaf_level[i] - 1; l >= 0; --l) {
      for (int j = 0; j < dim; ++j) g[j] >>= 1;
      u64 key = morton(dim, g);
      if (!R[l].insert(key)) break;
      work.push_back({l, key});
    }
  }
  i64 added = close_balance(dim, dom, R, work);
  GMG_REQUIRE(added == 0 || (flags & GMG_CLOSE_BALANCE), GMG_E_UNBALANCED,
              "forest violates 2:1 vertex balance");
  return forest_from_refined(dim, trees, R);
}

}  // namespace gmg

namespace gmg {

// Number of distinct Q_k nodes of all leaves (reading R22: "DoFs" = all leaf
// nodes, hanging and Dirichlet included) without building the topology: the
// finest node lattice is cut into slabs along x; each slab gathers the node keys
// of the leaves meeting it that fall into its half-open x range, sorts and counts
// the distinct ones.  Memory ~ (all node occurrences) / n_slabs, so config-5
// forests of 0.25-1B nodes can be counted on a small host.
i64 count_leaf_nodes(const Forest& f, int k) {
  GMG_REQUIRE(k >= 1 && k <= 4, GMG_E_INVALID_ARG, "k");
  const int d = f.dim, L = f.L;
  const i64 X = (i64)k * f.ext[0] << L;                 // lattice points 0..X along x
  const i64 n_leaves = f.n_leaves();
  int nn = 1;
  for (int j = 0; j < d; ++j) nn *= k + 1;
  const i64 occ = n_leaves * nn;
  const i64 target = 1 << 26;                           // ~64M keys (0.5 GB) per slab
  i64 n_slabs = std::max<i64>(1, std::min<i64>(X + 1, (occ + target - 1) / target));
  const i64 emax = std::max({f.ext[0], f.ext[1], f.ext[2]});
  const int cbits = bits_for((u64)(k * emax) << L);
  GMG_REQUIRE(cbits * d <= 64, GMG_E_DEPTH, "lattice keys exceed 64 bits");
  i64 total = 0;
  std::vector<u64> keys;
  for (i64 sl = 0; sl < n_slabs; ++sl) {
    const i64 x0 = (X + 1) * sl / n_slabs, x1 = (X + 1) * (sl + 1) / n_slabs;   // [x0, x1)
    keys.clear();
    for (i64 i = 0; i < n_leaves; ++i) {
      const int l = f.level[i];
      const i64 sh = L - l;
      const i64 lo = ((i64)k * f.gc[i][0]) << sh, hi = lo + ((i64)k << sh);
      if (hi < x0 || lo >= x1) continue;
      for (int b = 0; b < nn; ++b) {
        Vec3 P{0, 0, 0};
        int r = b;
        for (int j = 0; j < d; ++j) {
          P[j] = ((i64)k * f.gc[i][j] + r % (k + 1)) << sh;
          r /= (k + 1);
        }
        if (P[0] < x0 || P[0] >= x1) continue;
        keys.push_back(morton(d, P));
      }
    }
    radix_sort_keys(keys, cbits * d);
    for (size_t q = 0; q < keys.size(); ++q)
      if (q == 0 || keys[q] != keys[q - 1]) ++total;
  }
  return total;
}

}  // namespace gmg
