// Device order of the rank-local level vectors and the chunk tables of the
// fused level-operator kernels (host, integer).
//
// A chunk is CH_F consecutive local families of level l (SFC order).  The owned
// DoFs of a level are renumbered on the device as
//     [ R1 | R2 | R3 | ghosts ]
//   R1  DoFs touched by the families of exactly one chunk and by no other rank,
//       grouped by that chunk (contiguous per chunk, Morton order inside): the
//       chunk's CTA sees every contribution to them, so it finishes the operator
//       row and applies the Chebyshev / residual update in its epilogue;
//   R2  the other owned DoFs touched only locally (shared by >= 2 chunks), whose
//       rows are completed by fp64 reductions in L2 and finished by a streaming
//       pass over [r2_begin, r3_begin);
//   R3  owned DoFs another rank needs (its families touch them or it prolongates
//       from them), finished after the ghost export-add;
//   ghosts keep their order (the exchange plans address them by position).
// Level 0 keeps the identity order (no families, dense coarse solve).
// The renumbering is internal to the device layer: the integer exports use the
// global (owner, Morton) order of the paper's numbering, and the
// single-operator entry points permute at the boundary.
#pragma once

#include "forest.hpp"

namespace gmg {

constexpr int CH_F = 8;          // families per chunk (= warps per CTA of the fused kernels)
constexpr uint16_t LOC_NONE = 0xFFFF;

// Chunk-local shared-memory slots: the R1 range [r1_off, r1_off + n_r1) is
// staged by one bulk copy of the 16-byte aligned span starting at r1_off & ~1,
// so R1 DoF i sits in slot i + (r1_off & 1); halo DoF j sits in slot n_r1 + 2 + j.
struct ChunkLevel {
  i64 n_chunks = 0;
  i64 n_r1 = 0, r2_begin = 0, r3_begin = 0, n_owned = 0;
  int max_slots = 0;                     // max over chunks of n_r1 + 2 + n_halo
  int max_r1 = 0, max_halo = 0;
  std::vector<i32> meta;                 // [n_chunks][4]: r1_off, n_r1, halo_off, n_halo
  std::vector<i32> halo;                 // device-local DoF of each halo slot
  std::vector<uint16_t> loc;             // [n_chunks * CH_F][(2k+1)^d] slot, LOC_NONE = Dirichlet
};

struct DevicePlan {
  std::vector<std::vector<i32>> perm;    // per level: rank-local index -> device index
  std::vector<ChunkLevel> lv;
};

// Computes the device order from T's tables and rewrites T in place (every
// local DoF index of every table is mapped through perm).
DevicePlan plan_device_order(LocalTopo& T);

}  // namespace gmg
