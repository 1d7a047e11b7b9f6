// Family-patch geometry and the boundary test shared by the global and the
// rank-local topology builders (host, integer).
#pragma once

#include "forest.hpp"

namespace gmg {

struct PatchTables {
  int d, k, n1p, np, nn, nch, ndir;
  std::vector<std::array<int, 3>> pa;  // patch node coordinates
  std::vector<uint8_t> childmask;      // children whose closure contains patch node a
  std::vector<u32> dirmask;            // neighbour directions whose shared region contains a
  std::vector<std::vector<int>> cell_to_patch;  // [child][local b] -> patch a
  PatchTables(int d_, int k_) : d(d_), k(k_) {
    n1p = 2 * k + 1;
    np = 1, nn = 1;
    for (int j = 0; j < d; ++j) { np *= n1p; nn *= (k + 1); }
    nch = 1 << d;
    ndir = d == 2 ? 9 : 27;
    pa.resize(np);
    childmask.resize(np);
    dirmask.resize(np);
    for (int a = 0; a < np; ++a) {
      int r = a;
      for (int j = 0; j < 3; ++j) {
        pa[a][j] = j < d ? r % n1p : 0;
        if (j < d) r /= n1p;
      }
      uint8_t cm = 0;
      for (int c = 0; c < nch; ++c) {
        bool in = true;
        for (int j = 0; j < d; ++j) {
          int cj = (c >> j) & 1;
          if (cj == 0 && pa[a][j] > k) in = false;
          if (cj == 1 && pa[a][j] < k) in = false;
        }
        if (in) cm |= (uint8_t)(1u << c);
      }
      childmask[a] = cm;
      u32 dm = 0;
      for (int o = 0; o < ndir; ++o) {
        int off[3] = {o % 3 - 1, (o / 3) % 3 - 1, d == 3 ? o / 9 - 1 : 0};
        if (off[0] == 0 && off[1] == 0 && off[2] == 0) continue;
        bool in = true;
        for (int j = 0; j < d; ++j) {
          if (off[j] == -1 && pa[a][j] != 0) in = false;
          if (off[j] == 1 && pa[a][j] != 2 * k) in = false;
        }
        if (in) dm |= 1u << o;
      }
      dirmask[a] = dm;
    }
    cell_to_patch.assign(nch, std::vector<int>(nn));
    for (int c = 0; c < nch; ++c)
      for (int b = 0; b < nn; ++b) {
        int r = b, a = 0, mul = 1;
        for (int j = 0; j < d; ++j) {
          int bj = r % (k + 1);
          r /= (k + 1);
          a += (((c >> j) & 1) * k + bj) * mul;
          mul *= n1p;
        }
        cell_to_patch[c][b] = a;
      }
  }
};

inline bool on_boundary(const Forest& f, int k, const Vec3& X) {
  // x on the boundary <=> some x + eps*s lies outside every tree
  const i64 T = (i64)k << f.L;
  for (int c = 0; c < (1 << f.dim); ++c) {
    Vec3 tp{0, 0, 0};
    for (int j = 0; j < f.dim; ++j) {
      i64 v = ((c >> j) & 1) ? X[j] : X[j] - 1;
      tp[j] = v >= 0 ? v / T : -1;
    }
    bool inside = true;
    for (int j = 0; j < f.dim; ++j)
      if (tp[j] < 0 || tp[j] >= f.ext[j]) inside = false;
    if (inside && !f.occ[(size_t)((tp[2] * f.ext[1] + tp[1]) * f.ext[0] + tp[0])]) inside = false;
    if (!inside) return true;
  }
  return false;
}


enum : uint8_t { F_B = 1, F_EREG = 2, F_LEAF = 4 };

}  // namespace gmg
