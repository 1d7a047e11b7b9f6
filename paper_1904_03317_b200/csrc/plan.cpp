// Device order and chunk tables (see plan.hpp).
#include "plan.hpp"

#include <climits>

namespace gmg {

static inline i64 dec(i32 v) { return v >= 0 ? (i64)v : (v <= -2 ? -2 - (i64)v : -1); }
static inline i32 remap_enc(i32 v, const std::vector<i32>& p) {
  if (v >= 0) return p[v];
  if (v <= -2) return -2 - p[-2 - (i64)v];
  return -1;
}

DevicePlan plan_device_order(LocalTopo& T) {
  const int d = T.dim, k = T.k, L = T.L, F = CH_F;
  int nn = 1, np = 1;
  for (int j = 0; j < d; ++j) {
    nn *= k + 1;
    np *= 2 * k + 1;
  }
  DevicePlan P;
  P.perm.resize(L + 1);
  P.lv.resize(L + 1);
  // ---------------- 1. device order of every level (from the original tables)
  for (int l = 0; l <= L; ++l) {
    const LocalLevel& v = T.lv[l];
    const i64 n = v.n_local(), no = v.n_owned;
    ChunkLevel& C = P.lv[l];
    std::vector<i32>& perm = P.perm[l];
    perm.resize(n);
    C.n_owned = no;
    if (l == 0 || v.n_fam == 0) {
      for (i64 i = 0; i < n; ++i) perm[i] = (i32)i;
      C.r2_begin = 0;          // identity order: the streaming passes cover every owned DoF
      C.r3_begin = no;
      continue;
    }
    const i64 nch = (v.n_fam + F - 1) / F;
    C.n_chunks = nch;
    std::vector<i32> first(n, INT_MAX), last(n, -1);
    for (i64 f = 0; f < v.n_fam; ++f) {
      const i32 c = (i32)(f / F);
      for (int a = 0; a < np; ++a) {
        const i64 g = dec(v.fam_dofs[(size_t)f * np + a]);
        if (g < 0) continue;
        first[g] = std::min(first[g], c);
        last[g] = std::max(last[g], c);
      }
    }
    std::vector<char> remote(no, 0);
    for (i32 s : v.send_idx) remote[s] = 1;
    auto is_r1 = [&](i64 i) { return i < no && !remote[i] && last[i] >= 0 && first[i] == last[i]; };
    std::vector<i64> start(nch + 1, 0);
    for (i64 i = 0; i < no; ++i)
      if (is_r1(i)) start[first[i] + 1]++;
    for (i64 c = 0; c < nch; ++c) start[c + 1] += start[c];
    C.n_r1 = start[nch];
    std::vector<i64> fill(start.begin(), start.end() - 1);
    i64 pos = C.n_r1;
    for (i64 i = 0; i < no; ++i) {
      if (is_r1(i)) perm[i] = (i32)fill[first[i]]++;
    }
    C.r2_begin = C.n_r1;
    for (i64 i = 0; i < no; ++i)
      if (!is_r1(i) && !remote[i]) perm[i] = (i32)pos++;
    C.r3_begin = pos;
    for (i64 i = 0; i < no; ++i)
      if (remote[i]) perm[i] = (i32)pos++;
    GMG_REQUIRE(pos == no, GMG_E_STATE, "device order is not a permutation");
    for (i64 i = no; i < n; ++i) perm[i] = (i32)i;
    // ---------------- chunk tables
    C.meta.resize((size_t)nch * 4);
    C.loc.assign((size_t)nch * F * np, LOC_NONE);   // whole chunks: one aligned bulk copy each
    std::vector<i32> hl;
    for (i64 c = 0; c < nch; ++c) {
      const i64 f0 = c * F, f1 = std::min<i64>(v.n_fam, f0 + F);
      const i64 r1 = start[c], n1 = start[c + 1] - start[c];
      hl.clear();
      for (i64 f = f0; f < f1; ++f)
        for (int a = 0; a < np; ++a) {
          const i64 g = dec(v.fam_dofs[(size_t)f * np + a]);
          if (g >= 0 && !(is_r1(g) && first[g] == c)) hl.push_back(perm[g]);
        }
      std::sort(hl.begin(), hl.end());
      hl.erase(std::unique(hl.begin(), hl.end()), hl.end());
      const i64 nslot = n1 + 2 + (i64)hl.size();
      GMG_REQUIRE(nslot <= (i64)F * np + 2 && nslot < LOC_NONE, GMG_E_STATE, "chunk too large");
      C.max_slots = std::max<int>(C.max_slots, (int)nslot);
      C.max_r1 = std::max<int>(C.max_r1, (int)n1);
      C.max_halo = std::max<int>(C.max_halo, (int)hl.size());
      const i64 sh = r1 & 1;
      C.meta[(size_t)c * 4 + 0] = (i32)r1;
      C.meta[(size_t)c * 4 + 1] = (i32)n1;
      C.meta[(size_t)c * 4 + 2] = (i32)C.halo.size();
      C.meta[(size_t)c * 4 + 3] = (i32)hl.size();
      for (i64 f = f0; f < f1; ++f)
        for (int a = 0; a < np; ++a) {
          const i64 g = dec(v.fam_dofs[(size_t)f * np + a]);
          if (g < 0) continue;
          const i64 p = perm[g];
          uint16_t s;
          if (p >= r1 && p < r1 + n1) s = (uint16_t)(p - r1 + sh);
          else s = (uint16_t)(n1 + 2 + (std::lower_bound(hl.begin(), hl.end(), (i32)p) - hl.begin()));
          C.loc[(size_t)f * np + a] = s;
        }
      C.halo.insert(C.halo.end(), hl.begin(), hl.end());
    }
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
