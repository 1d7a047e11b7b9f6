// Device order of the rank-local level vectors (host, integer).
//
// On levels with families the owned DoFs are renumbered on the device as
//     [ R1 | rest of the owned DoFs | ghosts ]
//   R1  the owned DoFs that exactly one local family patch touches and that no
//       other rank needs: every patch-interior node ((2k+1)^d patch positions
//       with every coordinate in 1 .. 2k-1) and the patch-boundary nodes with
//       no neighbouring family on the level (61 % of c3's finest level rows
//       against 34 % patch-interior: the level is a thin shell).  The
//       level-operator kernel holds their complete row, stores it instead of
//       reducing it, and finishes the Chebyshev step on them in its epilogue
//       (kernels.cuh, fam_tensor_apply<..., CHEB>); grouped by family (SFC
//       order), patch order (z-major) inside the family;
//   the rest keep their (owner, Morton) order and are finished by the streaming
//   Chebyshev pass over [n_r1, n_pad).
// Where 8 consecutive local families form a complete grandfamily (their parents
// are the 8 children of one level-(l-2) cell, one coefficient) the operator runs
// on the grandfamily's (4k+1)^3 patch instead (gfam_tensor_apply): "patch" above
// then means the executed patch -- R1 counts the patches that touch a DoF and
// orders R1 by executed patch (SFC order of its first family), patch order inside.
// GMG_GFAM=0 turns grandfamily patches off.
// Level 0 keeps the identity order.  The renumbering is internal to the device
// layer: integer exports use the global order of the paper's numbering
// and the single-operator entry points permute at the boundary.
#pragma once

#include "forest.hpp"

namespace gmg {

struct DevicePlan {
  std::vector<std::vector<i32>> perm;    // per level: rank-local index -> device index
  std::vector<i64> n_r1;                 // per level: R1 = device indices [0, n_r1)
  // grandfamily patches (3D Q2 tensor levels, kernels.cuh gfam_tensor_apply): per
  // level the table [n_gf][GF_ROW] in device order, the coefficient per grandfamily
  // (config 4; empty = 1) and the families NOT in a grandfamily (run by the family
  // kernel through a list); singles is empty and n_gf = 0 where grandfamilies are off
  std::vector<i64> n_gf;
  std::vector<std::vector<i32>> gx, singles;
  std::vector<std::vector<i32>> gr1;     // per grandfamily: (first R1 row, R1 rows) -- contiguous by construction
  // n_ranks > 1: executed patches split into interior (no ghost node: can run while
  // the ghost import is in flight) and boundary ones -- family indices (over the
  // families the family kernel runs) and grandfamily indices; empty for one rank
  std::vector<std::vector<i32>> fam_int, fam_bnd, gf_int, gf_bnd;
  std::vector<std::vector<double>> gcoef;
};

// Computes the device order from T's tables and rewrites T in place (every
// local DoF index of every table is mapped through perm).
DevicePlan plan_device_order(LocalTopo& T, bool grandfamilies = true, int gf_min_level = 2);

}  // namespace gmg
