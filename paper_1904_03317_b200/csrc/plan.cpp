// Device order of the level vectors (see plan.hpp).
#include "plan.hpp"

namespace gmg {

static inline i64 dec(i32 v) { return v >= 0 ? (i64)v : (v <= -2 ? -2 - (i64)v : -1); }
static inline i32 remap_enc(i32 v, const std::vector<i32>& p) {
  if (v >= 0) return p[v];
  if (v <= -2) return -2 - p[-2 - (i64)v];
  return -1;
}

DevicePlan plan_device_order(LocalTopo& T) {
  const int d = T.dim, k = T.k, L = T.L;
  const int NP1 = 2 * k + 1;
  int nn = 1, np = 1;
  for (int j = 0; j < d; ++j) {
    nn *= k + 1;
    np *= NP1;
  }
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
      // number of local family patches touching each local DoF
      std::vector<uint8_t> touch(n, 0);
      for (i64 f = 0; f < v.n_fam; ++f)
        for (int a = 0; a < np; ++a) {
          const i64 g = dec(v.fam_dofs[(size_t)f * np + a]);
          if (g >= 0 && touch[g] < 255) ++touch[g];
        }
      for (i64 f = 0; f < v.n_fam; ++f) {
        for (int a : inner)
          GMG_REQUIRE(dec(v.fam_dofs[(size_t)f * np + a]) >= 0, GMG_E_STATE, "interior patch node without a DoF");
        for (int a = 0; a < np; ++a) {
          const i64 g = dec(v.fam_dofs[(size_t)f * np + a]);
          if (g >= 0 && g < no && touch[g] == 1 && !remote[g] && perm[g] < 0) perm[g] = (i32)pos++;
        }
      }
      P.n_r1[l] = pos;
      // the rest in the order the family patches first reach them (patch order)
      for (i64 f = 0; f < v.n_fam; ++f)
        for (int a = 0; a < np; ++a) {
          const i64 g = dec(v.fam_dofs[(size_t)f * np + a]);
          if (g >= 0 && g < no && perm[g] < 0) perm[g] = (i32)pos++;
        }
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
    for (auto& e : v.fam_dofs) e = remap_enc(e, p);
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
  return P;
}

}  // namespace gmg
