// Variable coefficient of config 4 (BASELINE configs[3]): a piecewise-constant
// a per level-2 cell.  The bilinear form on every level is the restriction of
// a(u, v) = int a grad u . grad v, so
//  * a cell of level >= 2 lies inside one level-2 cell: A_T = a * A_T(1);
//    the 2^d children of a level->=3 family share the coefficient;
//  * a cell of level 0 or 1 covers (2^(2-l))^d level-2 sub-boxes: A_T is the
//    exact integral over the sub-boxes, a sum of Kronecker terms of the 1-D
//    stiffness / mass matrices of the cell's basis restricted to each
//    sub-interval (reading R15 of DESIGN.md).
#include <cmath>

#include "forest.hpp"

namespace gmg {

namespace {
// 1-D Lagrange basis of degree k on the equidistant nodes a/k of [0,1]
double lag(int k, int a, double t) {
  double v = 1.0;
  for (int b = 0; b <= k; ++b)
    if (b != a) v *= (t - (double)b / k) / ((double)(a - b) / k);
  return v;
}
double lag_d(int k, int a, double t) {
  double s = 0.0;
  for (int c = 0; c <= k; ++c) {
    if (c == a) continue;
    double v = 1.0 / ((double)(a - c) / k);
    for (int b = 0; b <= k; ++b)
      if (b != a && b != c) v *= (t - (double)b / k) / ((double)(a - b) / k);
    s += v;
  }
  return s;
}
// stiffness / mass of the basis over [lo, hi] (3-point Gauss-Legendre: exact to degree 5 >= 2k)
void sub_matrices(int k, double lo, double hi, std::vector<double>& Km, std::vector<double>& Mm) {
  const double gx[3] = {-std::sqrt(0.6), 0.0, std::sqrt(0.6)}, gw[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
  const int n = k + 1;
  Km.assign(n * n, 0.0);
  Mm.assign(n * n, 0.0);
  for (int q = 0; q < 3; ++q) {
    const double t = lo + (hi - lo) * 0.5 * (gx[q] + 1.0), w = gw[q] * 0.5 * (hi - lo);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        Km[i * n + j] += w * lag_d(k, i, t) * lag_d(k, j, t);
        Mm[i * n + j] += w * lag(k, i, t) * lag(k, j, t);
      }
  }
}
}  // namespace

void attach_coefficients(LocalTopo& Lt, const Forest& f, const Partition& p, const double* coef2) {
  if (!coef2) return;
  const int d = Lt.dim, k = Lt.k, nch = 1 << d;
  GMG_REQUIRE(Lt.L >= 2, GMG_E_INVALID_ARG, "coefficient per level-2 cell needs >= 3 levels");
  const std::vector<u64>& key2 = p.levels[2].key;
  auto coef_of_key2 = [&](u64 key) {
    auto it = std::lower_bound(key2.begin(), key2.end(), key);
    GMG_REQUIRE(it != key2.end() && *it == key, GMG_E_STATE, "level-2 ancestor not found");
    const double a = coef2[it - key2.begin()];
    GMG_REQUIRE(a > 0 && std::isfinite(a), GMG_E_INVALID_ARG, "coefficient must be positive and finite");
    return a;
  };
  const int n1 = k + 1, nn = d == 3 ? n1 * n1 * n1 : n1 * n1;
  for (int l = 0; l <= Lt.L; ++l) {
    LocalLevel& v = Lt.lv[l];
    const std::vector<u64>& keys = p.levels[l].key;
    if (l >= 2) {
      v.cell_coef.resize(v.n_cells);
      for (i64 c = 0; c < v.n_cells; ++c) v.cell_coef[c] = coef_of_key2(keys[v.cell_global[c]] >> (d * (l - 2)));
      if (l >= 3) {
        v.fam_coef.resize(v.n_fam);
        for (i64 fm = 0; fm < v.n_fam; ++fm) {
          v.fam_coef[fm] = v.cell_coef[fm * nch];
          for (int c = 1; c < nch; ++c)
            GMG_REQUIRE(v.cell_coef[fm * nch + c] == v.fam_coef[fm], GMG_E_STATE, "family spans two coefficients");
        }
      }
      continue;
    }
    // levels 0, 1: exact sub-box element matrices
    const int nsub = 1 << (2 - l);
    std::vector<std::vector<double>> Ks(nsub), Ms(nsub);
    for (int s = 0; s < nsub; ++s) sub_matrices(k, (double)s / nsub, (double)(s + 1) / nsub, Ks[s], Ms[s]);
    const double hs = d == 3 ? std::ldexp(1.0, -l) : 1.0;   // h^(d-2)
    v.cell_elem.assign((size_t)v.n_cells * nn * nn, 0.0);
    const int nsb = d == 3 ? nsub * nsub * nsub : nsub * nsub;
    for (i64 c = 0; c < v.n_cells; ++c) {
      const Vec3 G = unmorton(d, keys[v.cell_global[c]]);
      double* A = v.cell_elem.data() + (size_t)c * nn * nn;
      for (int sb = 0; sb < nsb; ++sb) {
        const int sv[3] = {sb % nsub, (sb / nsub) % nsub, d == 3 ? sb / (nsub * nsub) : 0};
        Vec3 G2{0, 0, 0};
        for (int j = 0; j < d; ++j) G2[j] = G[j] * nsub + sv[j];
        const double a = coef_of_key2(morton(d, G2));
        for (int b = 0; b < nn; ++b)
          for (int b2 = 0; b2 < nn; ++b2) {
            const int bi[3] = {b % n1, (b / n1) % n1, b / (n1 * n1)};
            const int bj[3] = {b2 % n1, (b2 / n1) % n1, b2 / (n1 * n1)};
            double sum = 0.0;
            for (int i = 0; i < d; ++i) {
              double prod = 1.0;
              for (int j = 0; j < d; ++j) {
                const std::vector<double>& m = (j == i) ? Ks[sv[j]] : Ms[sv[j]];
                prod *= m[bi[j] * n1 + bj[j]];
              }
              sum += prod;
            }
            A[(size_t)b * nn + b2] += a * hs * sum;
          }
      }
    }
  }
}

}  // namespace gmg
