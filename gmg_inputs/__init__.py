"""Seeded synthetic inputs shared by the oracle (``oracle/``) and the CUDA path.

This module holds NO arithmetic of the method (no forest rule, no FEM, no
multigrid).  It only provides

* a counter-based splitmix64 generator (SURVEY.md §8(d) "Synthetic inputs":
  seed 190403317, uniform u = (z >> 11) * 2^-53, v = 2u - 1 in [-1, 1),
  log-uniform coefficient a = 10^(4u - 2));
* the configuration table: plain parameters of the five BASELINE.json
  configs (dimension, degree, brick of trees, refinement-recipe parameters as
  exact integers/rationals).  The refinement *predicates* themselves are
  implemented independently on both sides (oracle/forest.py and the C++
  library), see DESIGN.md "Input recipe".

Both sides draw random values by **canonical index** (the p = 1 ordering), so
results are independent of the number of ranks.
"""
from __future__ import annotations

import numpy as np

SEED = 190403317
GAMMA = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1

# stream ids
STREAM_RHS = 1          # c1 right-hand side over canonical free leaf DoFs
STREAM_COEF = 2         # c4 per-level-2-cell coefficient
STREAM_PROBE = 3        # random probe vectors for parity tests


def splitmix64(seed: int, stream: int, index) -> np.ndarray:
    """Counter-based splitmix64: value number ``index`` of ``stream``.

    state = seed + (stream << 32) * GAMMA + (index + 1) * GAMMA  (mod 2^64),
    followed by the splitmix64 output finaliser.
    """
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = np.uint64((seed + ((stream << 32) * GAMMA)) & _M64)
        z = base + (idx + np.uint64(1)) * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, stream: int, index) -> np.ndarray:
    """u = (z >> 11) * 2^-53 in [0, 1)."""
    z = splitmix64(seed, stream, index)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_pm1(n: int, stream: int = STREAM_RHS, seed: int = SEED, offset: int = 0) -> np.ndarray:
    """v = 2u - 1 in [-1, 1) for canonical indices offset .. offset+n-1."""
    return 2.0 * uniform01(seed, stream, np.arange(offset, offset + n, dtype=np.uint64)) - 1.0


def uniform_pm1_keys(keys, stream: int = STREAM_RHS, seed: int = SEED) -> np.ndarray:
    """v = 2u - 1 drawn by node key instead of canonical index (rank-local
    hierarchies: a rank knows the keys of its DoFs, not their canonical ranks);
    independent of the number of ranks."""
    return 2.0 * uniform01(seed, stream, np.asarray(keys, dtype=np.uint64)) - 1.0


def log_uniform_coef(n: int, stream: int = STREAM_COEF, seed: int = SEED) -> np.ndarray:
    """a = 10^(4u - 2), log-uniform in [1e-2, 1e2) (config 4)."""
    u = uniform01(seed, stream, np.arange(n, dtype=np.uint64))
    return np.power(10.0, 4.0 * u - 2.0)


# ---------------------------------------------------------------------------
# Configuration table (parameters only).  Distances/radii are exact rationals
# given as (numerator, denominator) in units of the tree edge length.
# ---------------------------------------------------------------------------
CONFIGS = {
    # BASELINE configs[0]: 2D Q1 on [0,1]^2; 4 global refinements; 3 passes
    # refining every leaf whose centre lies within 0.3 of the origin.
    "c1": dict(dim=2, k=1, trees=[(0, 0)], global_refinements=4,
               rule="center_ball", center=((0, 1), (0, 1)), radius=(3, 10), passes=3),
    # configs[1]: 2D L-shape [-1,1]^2 minus [0,1]^2, Q2, three trees in z-order
    # (0,0)=[-1,0]^2, (1,0)=[0,1]x[-1,0], (0,1)=[-1,0]x[0,1]; 3 global; refine
    # leaf T iff level(T) < 14 and dist(closure T, corner) <= 2^(6 - level),
    # to a fixed point (SURVEY c.2#18).  corner = brick point (1,1).
    "c2": dict(dim=2, k=2, trees=[(0, 0), (1, 0), (0, 1)], global_refinements=3,
               rule="corner_dist", corner=(1, 1), s=6, lmax=14, passes=None),
    # configs[2]: 3D [0,1]^3 Q2; 3 global; passes refining leaves whose closed
    # box meets the sphere |x - (1/2,1/2,1/2)| = 0.3 (min <= r <= max); P=7.
    "c3": dict(dim=3, k=2, trees=[(0, 0, 0)], global_refinements=3,
               rule="sphere_surface", center=((1, 2), (1, 2), (1, 2)), radius=(3, 10),
               shell=(0, 1), passes=7),
    # bounded samples of the c3 family (same recipe, fewer passes)
    "c3p2": dict(dim=3, k=2, trees=[(0, 0, 0)], global_refinements=3,
                 rule="sphere_surface", center=((1, 2), (1, 2), (1, 2)), radius=(3, 10),
                 shell=(0, 1), passes=2),
    "c3p4": dict(dim=3, k=2, trees=[(0, 0, 0)], global_refinements=3,
                 rule="sphere_surface", center=((1, 2), (1, 2), (1, 2)), radius=(3, 10),
                 shell=(0, 1), passes=4),
    # a 2x2x2 brick of trees (multi-cell coarse mesh: 27 free Q2 DoFs on level 0)
    # for the Chebyshev coarse solver; test case, not a BASELINE config
    "brick8": dict(dim=3, k=2, trees=[(x, y, z) for z in (0, 1) for y in (0, 1) for x in (0, 1)],
                   global_refinements=1, rule="sphere_surface", center=((1, 1), (1, 1), (1, 1)),
                   radius=(3, 5), shell=(0, 1), passes=2),
    # configs[3]: 3D variable coefficient, corner-graded toward (0,0,0)
    # (SURVEY c.2#20: dist(closure T, 0) <= 2^(s - level), level < lmax).  lmax
    # = 19 is the first value reaching ~100M leaf nodes (reading R20: 13,193,951
    # leaves, 107,140,241 nodes, 20 levels; lmax = 18 gives 99,063,795).
    "c4": dict(dim=3, k=2, trees=[(0, 0, 0)], global_refinements=3,
               rule="corner_dist", corner=(0, 0, 0), s=6, lmax=19, passes=None,
               coef="level2_log_uniform"),
    # configs[4]: the sphere-refined forest of config 3 scaled to ~125M DoFs per
    # GPU (reading R21): the 7 passes refine leaves meeting the closed shell
    # 0.3 - w <= |x - c| <= 0.3 + w, w = shell[0] / shell[1] the smallest multiple
    # of 2^-10 reaching 125M leaf nodes times the GPU count.  n = 1: w = 4/1024,
    # 125,785,013 nodes (w = 3/1024: 106,745,081).
    "c5": dict(dim=3, k=2, trees=[(0, 0, 0)], global_refinements=3,
               rule="sphere_surface", center=((1, 2), (1, 2), (1, 2)), radius=(3, 10),
               shell=(4, 1024), passes=7),
}

# config 5 for n GPUs: w_n / 2^-10, the smallest multiple giving >= 125M n leaf
# nodes, counted exactly (tools/count_c5.py -> profiles/c5_shell_counts.json):
# n = 1: 125,785,013 (m = 3: 106,745,081); n = 2: 258,586,909 (m = 10: 239,752,501);
# n = 4: 506,559,201 (m = 23: 487,502,405); n = 8: 1,008,420,977 (m = 49: 988,810,125).
C5_SHELL = {1: 4, 2: 11, 4: 24, 8: 50}


def config_c5(n_gpus: int) -> dict:
    cfg = dict(CONFIGS["c5"])
    cfg["shell"] = (C5_SHELL[n_gpus], 1024)
    return cfg


def config(name: str) -> dict:
    return dict(CONFIGS[name])
