"""Forest of refinement trees (oracle).  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §2.3: "the refinement procedure produces a tree
(or a forest, if M_0 consists of several cells) ... The level of such a cell is
its distance from its root cell"; refinement is isotropic bisection into 2^d
children; every refinement step is completed by a closure so that
"two leaf cells may only differ by one level, if they share a degree of
freedom" -- read as 2:1 balance over shared closure points
(vertex balance, reading R5).

Representation: a cell is (level, G) with G the integer *global brick*
coordinates of the cell on the level-l lattice of the brick of trees
(tree at brick position t covers G in [t*2^l, (t+1)*2^l)).  The SFC order
(p4est z-curve) is the Morton order of the global coordinates
scaled to a common finest level, x the fastest bit; with the trees' brick
positions interleaved as the top bits this is "tree order = z-order of the
brick positions, then Morton within the tree".
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def morton(coords: np.ndarray, nbits: int) -> np.ndarray:
    """Interleave the bits of integer coordinates [n, d]; x is the fastest bit."""
    c = np.asarray(coords, dtype=np.int64)
    n, d = c.shape
    key = np.zeros(n, dtype=np.int64)
    for b in range(nbits):
        for j in range(d):
            key |= ((c[:, j] >> b) & 1) << (b * d + j)
    return key


def nbits_for(maxval: int) -> int:
    return max(1, int(maxval).bit_length())


@dataclass
class Forest:
    dim: int
    trees: np.ndarray                 # [n_trees, dim] brick positions
    level: np.ndarray                 # [n_leaves] int64
    gc: np.ndarray                    # [n_leaves, dim] global coords at own level
    meta: dict = field(default_factory=dict)

    @property
    def n_leaves(self) -> int:
        return int(self.level.shape[0])

    @property
    def max_level(self) -> int:
        return int(self.level.max()) if self.n_leaves else 0

    def brick_extent(self) -> np.ndarray:
        return self.trees.max(axis=0) + 1

    def sfc_keys(self, L: int | None = None) -> np.ndarray:
        """Morton keys of the leaves' lower corners on the level-L lattice."""
        L = self.max_level if L is None else L
        fine = self.gc << (L - self.level)[:, None]
        nb = nbits_for(int(self.brick_extent().max()) << L)
        return morton(fine, nb)

    def sorted(self) -> "Forest":
        order = np.argsort(self.sfc_keys(), kind="stable")
        return Forest(self.dim, self.trees, self.level[order], self.gc[order], dict(self.meta))

    def tree_index(self) -> np.ndarray:
        """Tree id (position of the brick coordinate in z-order) of every leaf."""
        tpos = self.gc >> self.level[:, None]
        tkeys = morton(self.trees, nbits_for(int(self.trees.max()) + 1))
        tk = morton(tpos, nbits_for(int(self.trees.max()) + 1))
        order = np.argsort(tkeys)
        return order[np.searchsorted(tkeys[order], tk)]


def tree_order(trees) -> np.ndarray:
    """Trees sorted by the z-order of their brick positions."""
    t = np.asarray(trees, dtype=np.int64)
    k = morton(t, nbits_for(int(t.max()) + 1))
    return t[np.argsort(k)]


def in_domain(trees: np.ndarray, level: int | np.ndarray, gc: np.ndarray) -> np.ndarray:
    """True where the level-`level` lattice cell gc lies inside some tree."""
    tpos = gc >> int(level)
    ok = np.all(tpos >= 0, axis=1) & np.all(gc >= 0, axis=1)
    ext = trees.max(axis=0) + 1
    ok &= np.all(tpos < ext, axis=1)
    occ = np.zeros(tuple(ext), dtype=bool)
    occ[tuple(trees.T)] = True
    tp = np.clip(tpos, 0, ext - 1)
    ok &= occ[tuple(tp.T)]
    return ok


def coarse_forest(dim: int, trees) -> Forest:
    t = tree_order(trees)
    return Forest(dim, t, np.zeros(len(t), dtype=np.int64), t.copy())


def refine(f: Forest, mark: np.ndarray) -> Forest:
    """Replace every marked leaf by its 2^d children."""
    mark = np.asarray(mark, dtype=bool)
    keep_l = f.level[~mark]
    keep_g = f.gc[~mark]
    ml = f.level[mark]
    mg = f.gc[mark]
    kids_l = []
    kids_g = []
    for c in range(1 << f.dim):
        bits = np.array([(c >> j) & 1 for j in range(f.dim)], dtype=np.int64)
        kids_l.append(ml + 1)
        kids_g.append(2 * mg + bits)
    lev = np.concatenate([keep_l] + kids_l)
    gc = np.concatenate([keep_g] + kids_g).reshape(-1, f.dim)
    return Forest(f.dim, f.trees, lev, gc, dict(f.meta)).sorted()


def _lin(c: np.ndarray, R: int) -> np.ndarray:
    """Mixed-radix scalar key of integer points (coords in [-1, R-1))."""
    key = np.zeros(c.shape[0], dtype=np.int64)
    for j in range(c.shape[1] - 1, -1, -1):
        key = key * R + (c[:, j] + 1)
    return key


def balance_violators(f: Forest) -> np.ndarray:
    """Mask of leaves T whose closure contains a corner of a leaf U with
    level(U) >= level(T) + 2.  The 2:1 vertex balance of P:793-794 is violated
    exactly for such T: the intersection of the closures of a coarse cell and a
    smaller aligned dyadic cell always contains a corner of the smaller one."""
    L = f.max_level
    d = f.dim
    mark = np.zeros(f.n_leaves, dtype=bool)
    if L < 2:
        return mark
    R = (int(f.brick_extent().max()) << L) + 3
    corners = []
    for c in range(1 << d):
        bits = np.array([(c >> j) & 1 for j in range(d)], dtype=np.int64)
        corners.append((f.gc + bits) << (L - f.level)[:, None])
    corners = np.stack(corners, axis=1)                  # [n, 2^d, d]
    for lc in range(0, L - 1):
        leaves_here = np.nonzero(f.level == lc)[0]
        if leaves_here.size == 0:
            continue
        sel = f.level >= lc + 2
        if not sel.any():
            continue
        pk = np.unique(_lin(corners[sel].reshape(-1, d), R))
        # decode the unique points
        pts = np.empty((pk.size, d), dtype=np.int64)
        rem = pk.copy()
        for j in range(d):
            pts[:, j] = rem % R - 1
            rem //= R
        s = 1 << (L - lc)
        cand = []
        for c in range(1 << d):
            off = np.array([(c >> j) & 1 for j in range(d)], dtype=np.int64)
            # the level-lc cells whose closure contains the point
            cand.append(_lin(np.where(off == 0, pts // s, (pts - 1) // s), R))
        ck = np.unique(np.concatenate(cand))
        lk = _lin(f.gc[leaves_here], R)
        mark[leaves_here[np.isin(lk, ck)]] = True
    return mark


def close(f: Forest) -> Forest:
    """Closure to a fixed point: refine violators until none remain."""
    while True:
        m = balance_violators(f)
        if not m.any():
            return f
        f = refine(f, m)


# ---------------------------------------------------------------------------
# refinement predicates (integer arithmetic; reading R16: closed
# boxes, ties refine)
# ---------------------------------------------------------------------------

def _i64_guard(*arrs):
    for a in arrs:
        if a.size and float(np.abs(a).max()) > 2.0 ** 61:
            raise OverflowError("predicate arithmetic exceeds int64")


def _pred_center_ball(f: Forest, cfg) -> np.ndarray:
    """centre of the leaf within radius r of point c (c1):
    |(2G+1)/2^(l+1) - c|^2 <= r^2, multiplied through by (cd rd 2^(l+1))^2."""
    (rn, rd) = cfg["radius"]
    cen = cfg["center"]
    cd = 1
    for (_, d_) in cen:
        cd = int(np.lcm(cd, d_))
    scale = np.left_shift(np.int64(1), f.level + 1)          # 2^(l+1)
    tot = np.zeros(f.n_leaves, dtype=np.int64)
    for j in range(f.dim):
        cn, cdd = cen[j]
        num = (2 * f.gc[:, j] + 1) * cd - (cn * (cd // cdd)) * scale
        _i64_guard(num)
        tot = tot + num * num
    lhs = tot * (rd * rd)
    rhs = (rn * rn) * (scale * cd) * (scale * cd)
    _i64_guard(lhs.astype(np.float64), rhs.astype(np.float64))
    return lhs <= rhs


def _pred_sphere_surface(f: Forest, cfg) -> np.ndarray:
    """closed box meets the sphere |x - c| = r (c3): min|x-c| <= r <= max|x-c|;
    a shell half-width w widens this to min <= r + w and max >= r - w."""
    (rn, rd) = cfg["radius"]
    (wn, wd) = cfg.get("shell", (0, 1))
    cen = cfg["center"]
    cd = 1
    for (_, d_) in cen:
        cd = int(np.lcm(cd, d_))
    two_l = np.left_shift(np.int64(1), f.level)
    mn = np.zeros(f.n_leaves, dtype=np.int64)
    mx = np.zeros(f.n_leaves, dtype=np.int64)
    for j in range(f.dim):
        cn, cdd = cen[j]
        c = cn * (cd // cdd) * two_l          # centre in units 1/(cd 2^l)
        lo = f.gc[:, j] * cd
        hi = (f.gc[:, j] + 1) * cd
        a = lo - c
        b = c - hi
        dmin = np.maximum(np.maximum(a, b), 0)
        mn = mn + dmin * dmin
        mx = mx + np.maximum(a * a, b * b)
    den = rd * wd
    r_hi = rn * wd + wn * rd            # (r + w) * den
    r_lo = rn * wd - wn * rd            # (r - w) * den
    unit = cd * two_l
    lhs_min = mn * (den * den)
    rhs_hi = (r_hi * unit) * (r_hi * unit)
    _i64_guard(lhs_min.astype(np.float64), rhs_hi.astype(np.float64))
    cond_min = lhs_min <= rhs_hi
    if r_lo <= 0:
        cond_max = np.ones(f.n_leaves, dtype=bool)
    else:
        cond_max = mx * (den * den) >= (r_lo * unit) * (r_lo * unit)
    return cond_min & cond_max


def _pred_corner_dist(f: Forest, cfg) -> np.ndarray:
    """level < lmax and dist(closed box, corner) <= 2^(s - level) (c2, c4)."""
    corner = np.asarray(cfg["corner"], dtype=np.int64)
    s = cfg["s"]
    out = np.zeros(f.n_leaves, dtype=bool)
    for l in np.unique(f.level):
        sel = f.level == l
        c = corner << int(l)
        g = f.gc[sel]
        dv = np.maximum(np.maximum(g - c, c - (g + 1)), 0)
        d2 = (dv * dv).sum(axis=1)
        out[sel] = (l < cfg["lmax"]) & (d2 <= (1 << (2 * s)))
    return out


PREDICATES = {
    "center_ball": _pred_center_ball,
    "sphere_surface": _pred_sphere_surface,
    "corner_dist": _pred_corner_dist,
}


def generate(cfg: dict, passes: int | None = -1) -> Forest:
    """Build a config forest: global refinements, then refinement passes, each
    followed by the closure.  ``passes=None`` in the config means
    "repeat until no leaf is marked" (fixed point)."""
    f = coarse_forest(cfg["dim"], cfg["trees"])
    for _ in range(cfg["global_refinements"]):
        f = refine(f, np.ones(f.n_leaves, dtype=bool))
    npass = cfg["passes"] if passes == -1 else passes
    pred = PREDICATES[cfg["rule"]]
    it = 0
    while npass is None or it < npass:
        m = pred(f, cfg)
        if not m.any():
            break
        f = close(refine(f, m))
        it += 1
    f.meta["passes_done"] = it
    return f


def from_leaves(dim: int, trees, level, gc) -> Forest:
    return Forest(dim, tree_order(trees), np.asarray(level, dtype=np.int64),
                  np.asarray(gc, dtype=np.int64).reshape(-1, dim)).sorted()


# ---------------------------------------------------------------------------
# Mesh sequences of the partitioning study (§3.5, Fig. 3),
# one coarse cell read as [-1,1]^d (reading R27).  Every refinement
# step is followed by the closure.  A level-l cell G spans
# x_j in [2 G_j - 2^l, 2 G_j + 2 - 2^l] / 2^l; its centre is (2 G_j + 1 - 2^l) / 2^l.

def _centre2_times_4l(f: Forest) -> np.ndarray:
    """|centre|^2 * 4^level, exact in int64 for the small levels the tests use."""
    two_l = np.left_shift(np.int64(1), f.level)
    n = 2 * f.gc + 1 - two_l[:, None]
    _i64_guard(n.astype(np.float64) ** 2)
    return (n * n).sum(axis=1)


def sequence(dim: int, kind: str, L: int) -> Forest:
    """uniform: L global refinements.  circle: L times refine every leaf with a
    point inside the ball of radius 1/(4 pi) about the origin.  quadrant: one
    global refinement, then L-1 times refine the leaves of the negative
    quadrant [-1,0]^d.  annulus: L-3 global refinements, then refine the leaves
    whose centre lies in |x| <= 0.55, then 0.3 <= |x| <= 0.43, then
    0.335 <= |x| <= 0.39."""
    f = coarse_forest(dim, [tuple([0] * dim)])

    def step(mark):
        nonlocal f
        if mark.any():
            f = close(refine(f, mark))

    def all_leaves():
        return np.ones(f.n_leaves, dtype=bool)

    four_l = lambda: np.left_shift(np.int64(1), 2 * f.level)
    if kind == "uniform":
        for _ in range(L):
            step(all_leaves())
    elif kind == "circle":
        for _ in range(L):
            two_l = np.left_shift(np.int64(1), f.level)[:, None]
            lo = 2 * f.gc - two_l                      # box in units 2^-l
            hi = lo + 2
            v = np.where(lo > 0, lo, np.where(hi < 0, -hi, 0))
            d2 = (v * v).sum(axis=1).astype(np.float64)
            # distance < 1/(4 pi)  <=>  d2 / 4^l < 1 / (16 pi^2)
            step(d2 * (16.0 * np.pi ** 2) < four_l().astype(np.float64))
    elif kind == "quadrant":
        step(all_leaves())
        for _ in range(L - 1):
            two_l = np.left_shift(np.int64(1), f.level)[:, None]
            step(np.all(2 * f.gc + 2 - two_l <= 0, axis=1))
    elif kind == "annulus":
        if L < 4:
            raise ValueError("annulus needs L >= 4")
        for _ in range(L - 3):
            step(all_leaves())
        step(_centre2_times_4l(f) * 400 <= 121 * four_l())                       # r <= 0.55
        c2 = _centre2_times_4l(f)
        step((c2 * 100 >= 9 * four_l()) & (c2 * 10000 <= 1849 * four_l()))       # 0.3 .. 0.43
        c2 = _centre2_times_4l(f)
        step((c2 * 40000 >= 4489 * four_l()) & (c2 * 10000 <= 1521 * four_l()))  # 0.335 .. 0.39
    else:
        raise ValueError(kind)
    return f
