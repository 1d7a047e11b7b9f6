"""SFC partition, first-child rule and partition-efficiency model (oracle).
TEST INFRASTRUCTURE ONLY.

* Leaves are distributed "using a space filling curve": the SFC-sorted
  leaves are cut into n_p contiguous intervals, the first (N mod n_p) ranks get
  ceil(N/n_p) leaves (reading R4).
* "for each cell in the hierarchy, recursively assign the parent of a cell to
  the owner of the first child cell" -- implemented literally, bottom
  up, child 0 = lowest Morton child ("first (bottom-left) child").
* Model: N_l cells strictly on level l (reading R2), N_{l,p} of them
  owned by p; W_opt = (W_0 + sum_{l>=1} N_l)/n_p, W_sync = W_0 + sum_{l>=1}
  ceil(N_l/n_p), W_l = max_p N_{l,p}, W = W_0 + sum_{l>=1} W_l, eta = W_opt/W.
  Default (reading R3, as in the worked example P:699-711): level 0 is an
  ordinary level, i.e. W_0 enters W_opt as N_0, W_sync as ceil(N_0/n_p) and W
  as max_p N_{0,p}.  An override replaces all three by the given constant.
* Ghost children: level-l cells (l >= 1) whose owner differs from
  the owner of their parent.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from math import ceil

import numpy as np

from .forest import Forest, morton, nbits_for


def sfc_counts(n: int, p: int) -> np.ndarray:
    if p < 1:
        raise ValueError("n_ranks must be >= 1")
    base, rem = divmod(n, p)
    return np.array([base + 1 if r < rem else base for r in range(p)], dtype=np.int64)


def leaf_owners(f: Forest, p: int) -> np.ndarray:
    counts = sfc_counts(f.n_leaves, p)
    return np.repeat(np.arange(p, dtype=np.int64), counts)


@dataclass
class LevelCells:
    level: int
    gc: np.ndarray        # [n, d] sorted in SFC (Morton) order
    key: np.ndarray       # Morton keys (level lattice)
    is_leaf: np.ndarray   # bool
    owner: np.ndarray     # int64


def level_cells(f: Forest, leaf_owner: np.ndarray | None = None) -> list[LevelCells]:
    """C_l for l = 0..L: all cells of the forest with level exactly l (leaves and
    refined cells), with owners from the first-child rule."""
    L = f.max_level
    d = f.dim
    if leaf_owner is None:
        leaf_owner = np.zeros(f.n_leaves, dtype=np.int64)
    out: list[LevelCells] = [None] * (L + 1)
    # bottom-up: cells of level l = leaves of level l  U  parents of level l+1 cells
    child_gc = None
    for l in range(L, -1, -1):
        lsel = f.level == l
        gcs = [f.gc[lsel]]
        leaf = [np.ones(int(lsel.sum()), dtype=bool)]
        own = [leaf_owner[lsel]]
        if child_gc is not None and child_gc.gc.shape[0]:
            ch = child_gc
            first = np.all((ch.gc & 1) == 0, axis=1)          # child 0 of its parent
            pg = ch.gc[first] >> 1
            gcs.append(pg)
            leaf.append(np.zeros(pg.shape[0], dtype=bool))
            own.append(ch.owner[first])                      # owner of the first child
        gc = np.concatenate(gcs).reshape(-1, d)
        is_leaf = np.concatenate(leaf)
        owner = np.concatenate(own)
        nb = nbits_for(int(f.brick_extent().max()) << l)
        key = morton(gc, nb)
        o = np.argsort(key, kind="stable")
        lc = LevelCells(l, gc[o], key[o], is_leaf[o], owner[o])
        assert np.all(np.diff(lc.key) > 0), "duplicate cell"
        out[l] = lc
        child_gc = lc
    return out


@dataclass
class Model:
    N: np.ndarray          # [L+1]
    Nlp: np.ndarray        # [L+1, p]
    W_opt: Fraction
    W_sync: int
    W_l: np.ndarray
    W: int
    eta: Fraction


def model(cells: list[LevelCells], p: int, W0_override: int | None = None) -> Model:
    L = len(cells) - 1
    Nlp = np.zeros((L + 1, p), dtype=np.int64)
    for l, lc in enumerate(cells):
        Nlp[l] = np.bincount(lc.owner, minlength=p)[:p]
    N = Nlp.sum(axis=1)
    W_l = Nlp.max(axis=1)
    if W0_override is None:
        w0_opt, w0_sync, w0 = int(N[0]), ceil(Fraction(int(N[0]), p)), int(W_l[0])
    else:
        w0_opt = w0_sync = w0 = int(W0_override)
    W_opt = Fraction(w0_opt + int(N[1:].sum()), p)
    W_sync = w0_sync + sum(ceil(Fraction(int(n), p)) for n in N[1:])
    W = w0 + int(W_l[1:].sum())
    return Model(N, Nlp, W_opt, int(W_sync), W_l, int(W), W_opt / W)


def ghost_children(cells: list[LevelCells]) -> tuple[np.ndarray, np.ndarray]:
    """Per level l >= 1: (#cells whose owner != parent's owner, #cells)."""
    L = len(cells) - 1
    ghosts = np.zeros(L + 1, dtype=np.int64)
    total = np.zeros(L + 1, dtype=np.int64)
    for l in range(1, L + 1):
        ch = cells[l]
        par = cells[l - 1]
        nb = nbits_for(int(par.gc.max(initial=0)) + 1) + 1
        pk = morton(ch.gc >> 1, max(nb, nbits_for(int(ch.gc.max(initial=0)) + 1)))
        parkey = morton(par.gc, max(nb, nbits_for(int(ch.gc.max(initial=0)) + 1)))
        idx = np.searchsorted(parkey, pk)
        assert np.all(parkey[idx] == pk)
        ghosts[l] = int((ch.owner != par.owner[idx]).sum())
        total[l] = ch.gc.shape[0]
    return ghosts, total


def per_level_owners(cells: list[LevelCells], p: int) -> list[LevelCells]:
    """The alternative to the first-child rule that P:597 contrasts with (SURVEY
    §8(f) row 4, reading R29): each level partitioned on its own along
    the SFC, families (cells with a common parent; single cells on level 0) kept
    whole.  Written as a plain loop: a family whose first cell has index c among
    the N_l cells of level l goes to rank floor(p c / N_l)."""
    out = []
    for l, lc in enumerate(cells):
        n = lc.gc.shape[0]
        owner = np.empty(n, dtype=np.int64)
        c = 0
        while c < n:
            e = c + 1
            if l > 0:
                parent = tuple(lc.gc[c] >> 1)
                while e < n and tuple(lc.gc[e] >> 1) == parent:
                    e += 1
            owner[c:e] = (p * c) // n
            c = e
        out.append(LevelCells(lc.level, lc.gc, lc.key, lc.is_leaf, owner))
    return out
