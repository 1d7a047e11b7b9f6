// Device order of the level vectors (see plan.hpp).
#include "plan.hpp"

namespace gmg {

static inline i64 dec(i32 v) { return v >= 0 ? (i64)v : (v <= -2 ? -2 - (i64)v : -1); }
static inline i32 remap_enc(i32 v, const std::vector<i32>& p) {
  if (v >= 0) return p[v];
  if (v <= -2) return -2 - p[-2 - (i64)v];
  return -1;
}

// Node of grandfamily position (X, Y, Z) (0 .. 4k each) in family-patch terms:
// the family j = cx + 2 cy + 4 cz of the grandfamily and its patch position a.
static inline void gf_pos(int k, int X, int Y, int Z, int& j, int& a) {
  const int NP1 = 2 * k + 1;
  const int cx = X > 2 * k ? 1 : 0, cy = Y > 2 * k ? 1 : 0, cz = Z > 2 * k ? 1 : 0;
  j = cx + 2 * cy + 4 * cz;
  a = (X - 2 * k * cx) + NP1 * (Y - 2 * k * cy) + NP1 * NP1 * (Z - 2 * k * cz);
}

DevicePlan plan_device_order(LocalTopo& T, bool grandfamilies, int gf_min_level) {
  const int d = T.dim, k = T.k, L = T.L;
  const int NP1 = 2 * k + 1;
  int nn = 1, np = 1;
  for (int j = 0; j < d; ++j) {
    nn *= k + 1;
    np *= NP1;
  }
  const int G1 = 4 * k + 1, GNP = G1 * G1 * G1;
  const int xr = np + nn;   // xfer row: the family patch, then the parent's DoFs
  // interior patch positions, z-major (ascending patch index)
  std::vector<int> inner;
  for (int a = 0; a < np; ++a) {
    const int c[3] = {a % NP1, (a / NP1) % NP1, a / (NP1 * NP1)};
    bool in = true;
    for (int j = 0; j < d; ++j) in &= c[j] > 0 && c[j] < 2 * k;
    if (in) inner.push_back(a);
  }
  DevicePlan P;
  P.perm.resize(L + 1);
  P.n_r1.assign(L + 1, 0);
  P.n_gf.assign(L + 1, 0);
  P.gx.resize(L + 1);
  P.singles.resize(L + 1);
  P.gr1.resize(L + 1);
  for (auto* v : {&P.fam_int, &P.fam_bnd, &P.gf_int, &P.gf_bnd}) v->resize(L + 1);
  P.gcoef.resize(L + 1);
  // per level: grandfamilies in use (first local family of each) and a family ->
  // grandfamily map (-1: single)
  std::vector<std::vector<i32>> gfs(L + 1), fam_gf(L + 1);
  // ---------------- 1. device order of every level (from the original tables)
  for (int l = 0; l <= L; ++l) {
    const LocalLevel& v = T.lv[l];
    const i64 n = v.n_local(), no = v.n_owned;
    std::vector<i32>& perm = P.perm[l];
    perm.assign(n, -1);
    i64 pos = 0;
    // R1 only where the level operator runs fam_tensor_apply (3D; not on the
    // config-4 levels with per-cell coefficients or explicit element matrices)
    const bool tensor = d == 3 && l > 0 && v.n_fam > 0 && v.cell_elem.empty() &&
                        (v.cell_coef.empty() || !v.fam_coef.empty());
    if (tensor) {
      std::vector<char> remote(no, 0);
      for (i32 s : v.send_idx) remote[s] = 1;
      // grandfamily patches in use: Q2, one coefficient for all 8 families
      std::vector<i32>& fg = fam_gf[l];
      fg.assign(v.n_fam, -1);
      if (grandfamilies && k == 2 && l >= gf_min_level)
        for (i32 f0 : v.gf_first) {
          bool ok = true;
          if (!v.fam_coef.empty())
            for (int j = 1; j < 8; ++j) ok &= v.fam_coef[f0 + j] == v.fam_coef[f0];
          if (!ok) continue;
          for (int j = 0; j < 8; ++j) fg[f0 + j] = (i32)gfs[l].size();
          gfs[l].push_back(f0);
        }
      // executed patches in SFC order (a grandfamily at its first family), each
      // visiting its nodes in patch order, once per distinct node
      auto for_patches = [&](auto&& fn) {
        for (i64 f = 0; f < v.n_fam; ++f) {
          if (fg[f] < 0) {
            for (int a = 0; a < np; ++a) fn(dec(v.xfer[(size_t)f * xr + a]));
          } else if (gfs[l][fg[f]] == f) {
            for (int Z = 0; Z < G1; ++Z)
              for (int Y = 0; Y < G1; ++Y)
                for (int X = 0; X < G1; ++X) {
                  int j, a;
                  gf_pos(k, X, Y, Z, j, a);
                  fn(dec(v.xfer[(size_t)(f + j) * xr + a]));
                }
          }
        }
      };
      // number of executed patches touching each local DoF
      std::vector<uint8_t> touch(n, 0);
      for_patches([&](i64 g) {
        if (g >= 0 && touch[g] < 255) ++touch[g];
      });
      for (i64 f = 0; f < v.n_fam; ++f)
        for (int a : inner)
          GMG_REQUIRE(dec(v.xfer[(size_t)f * xr + a]) >= 0, GMG_E_STATE, "interior patch node without a DoF");
      for_patches([&](i64 g) {
        if (g >= 0 && g < no && touch[g] == 1 && !remote[g] && perm[g] < 0) perm[g] = (i32)pos++;
      });
      P.n_r1[l] = pos;
      // the rest in the order the executed patches first reach them (patch order)
      for_patches([&](i64 g) {
        if (g >= 0 && g < no && perm[g] < 0) perm[g] = (i32)pos++;
      });
    }
    for (i64 i = 0; i < no; ++i)
      if (perm[i] < 0) perm[i] = (i32)pos++;
    GMG_REQUIRE(pos == no, GMG_E_STATE, "device order is not a permutation");
    for (i64 i = no; i < n; ++i) perm[i] = (i32)i;
  }
  // ---------------- 2. rewrite the local tables in device order
  for (int l = 0; l <= L; ++l) {
    LocalLevel& v = T.lv[l];
    const std::vector<i32>& p = P.perm[l];
    const i64 n = v.n_local();
    for (auto& c : v.cell_dofs)
      if (c >= 0) c = p[c];
    if (l > 0) {
      const int row = np + nn;
      const std::vector<i32>& pc = P.perm[l - 1];
      for (i64 f = 0; f < v.n_fam; ++f) {
        i32* r = v.xfer.data() + (size_t)f * row;
        for (int a = 0; a < np; ++a) r[a] = remap_enc(r[a], p);
        for (int j = 0; j < nn; ++j)
          if (r[np + j] >= 0) r[np + j] = pc[r[np + j]];
      }
    }
    for (auto& s : v.send_idx) s = p[s];
    for (auto& s : v.recv_idx) s = p[s];
    std::vector<uint8_t> cls(n), lam(n);
    std::vector<double> ev(v.eig_v.size());
    for (i64 i = 0; i < n; ++i) {
      cls[p[i]] = v.cls[i];
      lam[p[i]] = v.lam[i];
      if (!ev.empty()) ev[p[i]] = v.eig_v[i];
    }
    v.cls.swap(cls);
    v.lam.swap(lam);
    v.eig_v.swap(ev);
  }
  for (size_t g = 0; g < T.leaf_local.size(); ++g)
    T.leaf_local[g] = P.perm[T.leaf_level[g]][T.leaf_local[g]];
  // ---------------- 3. grandfamily tables (device order) and the single families
  const int NCP = NP1 * NP1 * NP1, GROW = GNP + NCP;
  for (int l = 0; l <= L; ++l) {
    const LocalLevel& v = T.lv[l];
    if (gfs[l].empty()) continue;
    const std::vector<i32>& fg = fam_gf[l];
    P.n_gf[l] = (i64)gfs[l].size();
    std::vector<i32>& gx = P.gx[l];
    gx.assign((size_t)P.n_gf[l] * GROW, -1);
    for (size_t q = 0; q < gfs[l].size(); ++q) {
      const i64 f0 = gfs[l][q];
      i32* row = gx.data() + q * GROW;
      for (int Z = 0; Z < G1; ++Z)
        for (int Y = 0; Y < G1; ++Y)
          for (int X = 0; X < G1; ++X) {
            int j, a;
            gf_pos(k, X, Y, Z, j, a);
            const i64 g = dec(v.xfer[(size_t)(f0 + j) * xr + a]);
            // transfer owner inside the grandfamily: some family containing the node
            // holds it with a non-negative entry
            bool own = false;
            for (int cz = 0; cz < 2; ++cz)
              for (int cy = 0; cy < 2; ++cy)
                for (int cx = 0; cx < 2; ++cx) {
                  const int lx = X - 2 * k * cx, ly = Y - 2 * k * cy, lz = Z - 2 * k * cz;
                  if (lx < 0 || lx > 2 * k || ly < 0 || ly > 2 * k || lz < 0 || lz > 2 * k) continue;
                  const i32 e = v.xfer[(size_t)(f0 + cx + 2 * cy + 4 * cz) * xr + lx + NP1 * ly + NP1 * NP1 * lz];
                  if (e >= 0) own = true;
                }
            row[X + G1 * Y + G1 * G1 * Z] = g < 0 ? -1 : (own ? (i32)g : (i32)(-2 - g));
          }
      // G's family patch one level up: the 8 parents' (k+1)^3 nodes
      for (int c = 0; c < NP1; ++c)
        for (int b = 0; b < NP1; ++b)
          for (int a = 0; a < NP1; ++a) {
            const int cx = a > k ? 1 : 0, cy = b > k ? 1 : 0, cz = c > k ? 1 : 0;
            const int la = a - k * cx, lb = b - k * cy, lc = c - k * cz;
            const i32* xr = v.xfer.data() + (size_t)(f0 + cx + 2 * cy + 4 * cz) * (np + nn);
            row[GNP + a + NP1 * b + NP1 * NP1 * c] = xr[np + la + (k + 1) * lb + (k + 1) * (k + 1) * lc];
          }
      if (!v.fam_coef.empty()) P.gcoef[l].push_back(v.fam_coef[f0]);
      // R1 rows of this grandfamily: a contiguous run (R1 is ordered by executed patch)
      i32 lo = INT32_MAX, cntr = 0;
      for (int a = 0; a < GNP; ++a) {
        const i64 g = dec(row[a]);
        if (g >= 0 && g < P.n_r1[l]) {
          lo = std::min(lo, (i32)g);
          ++cntr;
        }
      }
      P.gr1[l].push_back(cntr ? lo : 0);
      P.gr1[l].push_back(cntr);
    }
    for (i64 f = 0; f < v.n_fam; ++f)
      if (fg[f] < 0) P.singles[l].push_back((i32)f);
  }
  // ---------------- interior / boundary patches (several ranks: overlap with the import)
  if (T.n_ranks > 1)
    for (int l = 1; l <= L; ++l) {
      const LocalLevel& v = T.lv[l];
      const bool tensor3 = d == 3 && v.n_fam > 0 && v.cell_elem.empty() && (v.cell_coef.empty() || !v.fam_coef.empty());
      if (!tensor3) continue;
      auto ghost_in = [&](const i32* row, int n) {
        for (int a = 0; a < n; ++a)
          if (dec(row[a]) >= v.n_owned) return true;
        return false;
      };
      const std::vector<i32>* fams = P.n_gf[l] > 0 ? &P.singles[l] : nullptr;
      const i64 nf = fams ? (i64)fams->size() : v.n_fam;
      for (i64 i = 0; i < nf; ++i) {
        const i64 f = fams ? (*fams)[i] : i;
        (ghost_in(v.xfer.data() + (size_t)f * xr, np) ? P.fam_bnd : P.fam_int)[l].push_back((i32)f);
      }
      for (i64 q = 0; q < P.n_gf[l]; ++q)
        (ghost_in(P.gx[l].data() + (size_t)q * GROW, GNP) ? P.gf_bnd : P.gf_int)[l].push_back((i32)q);
    }
  return P;
}

}  // namespace gmg
