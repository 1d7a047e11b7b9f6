"""Pins of the oracle's forest, closure, SFC partition and efficiency model
against what PAPER.md fixes (worked example P:669-718) and
brute-force enumerations (no GPU)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import forest as F
from oracle import partition as Pt
from gmg_inputs import config

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


# ---------------------------------------------------------------- brute force
def brute_balanced(f):
    """Every pair of leaves whose closures intersect differs by <= 1 level."""
    L = f.max_level
    lo = f.gc << (L - f.level)[:, None]
    hi = (f.gc + 1) << (L - f.level)[:, None]
    for i in range(f.n_leaves):
        touch = np.all((lo <= hi[i]) & (lo[i] <= hi), axis=1)
        if np.any(np.abs(f.level[touch] - f.level[i]) > 1):
            return False
    return True


def brute_dfs_order(f):
    """Depth-first traversal of the trees (children in x-fastest Morton order)."""
    leaves = {(int(l), tuple(int(v) for v in g)) for l, g in zip(f.level, f.gc)}
    out = []

    def rec(l, g):
        if (l, g) in leaves:
            out.append((l, g))
            return
        for c in range(1 << f.dim):
            rec(l + 1, tuple(2 * g[j] + ((c >> j) & 1) for j in range(f.dim)))

    for t in f.trees:
        rec(0, tuple(int(v) for v in t))
    return out


def brute_first_leaf_owner(f, owners):
    """owner(cell) = owner of the first SFC leaf in its subtree."""
    L = f.max_level
    res = {}
    lo = f.gc << (L - f.level)[:, None]
    keys = f.sfc_keys()
    for l in range(L + 1):
        for g in np.unique(f.gc[f.level >= l] >> (f.level[f.level >= l] - l)[:, None], axis=0):
            glo = g << (L - l)
            ghi = (g + 1) << (L - l)
            inside = np.all((lo >= glo) & (lo < ghi), axis=1)
            first = np.nonzero(inside)[0][np.argmin(keys[inside])]
            res[(l, tuple(int(v) for v in g))] = int(owners[first])
    return res


def fig2_forest(refined_child):
    f = F.coarse_forest(2, [(0, 0)])
    f = F.refine(f, np.ones(1, dtype=bool))
    m = np.zeros(4, dtype=bool)
    # leaves are in Morton order: child c at index c
    m[refined_child] = True
    return F.refine(f, m)


# ---------------------------------------------------------------- forest
def test_uniform_counts():
    for d in (2, 3):
        f = F.coarse_forest(d, [(0,) * d])
        for L in range(1, 4):
            f = F.refine(f, np.ones(f.n_leaves, dtype=bool))
            assert f.n_leaves == (1 << d) ** L


def test_corner_refinement_no_closure():
    # two uniform refinements, refine the corner leaf -> 19 leaves, balanced
    f = F.coarse_forest(2, [(0, 0)])
    f = F.refine(F.refine(f, [True]), np.ones(4, dtype=bool))
    m = np.zeros(16, dtype=bool)
    m[0] = True
    g = F.close(F.refine(f, m))
    assert g.n_leaves == 19 and brute_balanced(g)


def test_closure_triggers_and_is_minimal():
    # refine the corner twice more: the level-2 neighbours of a level-4 cell
    f = F.coarse_forest(2, [(0, 0)])
    f = F.refine(F.refine(f, [True]), np.ones(4, dtype=bool))
    m = np.zeros(f.n_leaves, dtype=bool)
    m[0] = True
    f = F.refine(f, m)                      # level-3 cells in the corner cell
    m = (f.level == 3) & np.all(f.gc == 1, axis=1)
    f = F.refine(f, m)                      # a level-4 cell touching level-2 leaves
    assert not brute_balanced(f)
    g = F.close(f)
    assert brute_balanced(g)
    # minimality: undoing any single closure-refinement family breaks balance
    assert F.close(g).n_leaves == g.n_leaves           # idempotence


@settings(max_examples=25, deadline=None)
@given(st.integers(2, 3), st.lists(st.integers(0, 10 ** 6), min_size=1, max_size=6),
       st.integers(0, 1))
def test_random_closure_balanced(d, picks, gref):
    f = F.coarse_forest(d, [(0,) * d])
    for _ in range(1 + gref):
        f = F.refine(f, np.ones(f.n_leaves, dtype=bool))
    for p in picks:
        m = np.zeros(f.n_leaves, dtype=bool)
        m[p % f.n_leaves] = True
        f = F.close(F.refine(f, m))
        if f.n_leaves > 600:
            break
    assert brute_balanced(f)
    # tiling: sum of leaf volumes equals the domain volume (integer)
    L = f.max_level
    assert int(np.sum(1 << (d * (L - f.level)))) == (1 << (d * L))
    # SFC order = depth-first traversal order
    dfs = brute_dfs_order(f)
    assert dfs == [(int(l), tuple(int(v) for v in g)) for l, g in zip(f.level, f.gc)]


def test_lshape_multitree_dfs_and_balance():
    cfg = dict(config("c2"))
    cfg["lmax"] = 6
    cfg["s"] = 1
    f = F.generate(cfg)
    assert brute_balanced(f)
    dfs = brute_dfs_order(f)
    assert dfs == [(int(l), tuple(int(v) for v in g)) for l, g in zip(f.level, f.gc)]


def test_config1_counts():
    g = gold("config_counts.json")["c1"]
    f = F.generate(config("c1"))
    assert f.n_leaves == g["leaves"]
    assert f.max_level + 1 == g["levels"]
    assert brute_balanced(f)


@pytest.mark.slow
def test_config2_counts():
    g = gold("config_counts.json")["c2"]
    f = F.generate(config("c2"))
    assert f.n_leaves == g["leaves"] and f.max_level + 1 == g["levels"]


# ---------------------------------------------------------------- partition
def test_sfc_counts_remainder():
    assert list(Pt.sfc_counts(7, 3)) == [3, 2, 2]
    assert list(Pt.sfc_counts(64, 4)) == [16] * 4
    with pytest.raises(ValueError):
        Pt.sfc_counts(5, 0)


@pytest.mark.parametrize("child", [0, 1, 2, 3])
def test_fig2_model_all_readings(child):
    """W_opt=3, W_sync=5, W=6, eta=1/2 -- holds for every choice of
    the refined level-1 cell (the figure is missing)."""
    gd = gold("fig2.json")
    f = fig2_forest(child)
    assert f.n_leaves == 7
    cells = Pt.level_cells(f, Pt.leaf_owners(f, 3))
    m = Pt.model(cells, 3)
    assert m.W_opt == Fraction(*gd["W_opt"])
    assert m.W_sync == gd["W_sync"]
    if child == 2:
        assert m.W == gd["W"] and m.eta == Fraction(*gd["eta"])


def test_fig2_reading_r1_details():
    gd = gold("fig2.json")
    f = fig2_forest(2)
    cells = Pt.level_cells(f, Pt.leaf_owners(f, 3))
    m = Pt.model(cells, 3)
    assert list(m.N) == gd["N"]
    assert list(m.Nlp[1]) == gd["N_lp_level1"]           # "#0 works on three cells", "#1 recuses itself"
    assert list(m.Nlp[2]) == gd["N_lp_level2"]
    assert cells[0].owner[0] == 0                         # "only processor #0 remains on the coarsest level"
    g, t = Pt.ghost_children(cells)
    assert list(g) == gd["ghost_children"] and list(t) == gd["children"]
    # parent of the four smallest cells is #0 because the first child is #0
    par = cells[1].owner[np.nonzero(~cells[1].is_leaf)[0][0]]
    assert par == 0


def test_uniform_model_S208():
    gd = gold("uniform_L2_p4.json")
    f = F.coarse_forest(2, [(0, 0)])
    for _ in range(2):
        f = F.refine(f, np.ones(f.n_leaves, dtype=bool))
    cells = Pt.level_cells(f, Pt.leaf_owners(f, 4))
    m = Pt.model(cells, 4)
    assert list(m.N) == gd["N"] and m.W == gd["W"]
    assert m.W_opt == Fraction(*gd["W_opt"]) and m.eta == Fraction(*gd["eta"])


def test_uniform_perfect_partition_P819():
    """p = 2^(d k) ranks: every level l >= k perfectly balanced."""
    for d in (2, 3):
        f = F.coarse_forest(d, [(0,) * d])
        for _ in range(3):
            f = F.refine(f, np.ones(f.n_leaves, dtype=bool))
        for kk in (1, 2):
            p = 1 << (d * kk)
            cells = Pt.level_cells(f, Pt.leaf_owners(f, p))
            m = Pt.model(cells, p)
            for l in range(kk, 4):
                assert m.W_l[l] * p == m.N[l]


@settings(max_examples=20, deadline=None)
@given(st.integers(2, 3), st.lists(st.integers(0, 10 ** 6), min_size=1, max_size=5),
       st.integers(1, 9))
def test_model_invariants_and_first_child(d, picks, p):
    f = F.coarse_forest(d, [(0,) * d])
    f = F.refine(f, np.ones(1, dtype=bool))
    for q in picks:
        m = np.zeros(f.n_leaves, dtype=bool)
        m[q % f.n_leaves] = True
        f = F.close(F.refine(f, m))
        if f.n_leaves > 300:
            break
    own = Pt.leaf_owners(f, p)
    cells = Pt.level_cells(f, own)
    m = Pt.model(cells, p)
    L = f.max_level
    # W >= W_sync >= W_opt, and they differ only by per-level rounding
    assert m.W >= m.W_sync >= m.W_opt
    assert m.W_sync - m.W_opt < L + 1
    assert 0 < m.eta <= 1
    if p == 1:
        assert m.eta == 1
    # independent tree walk: first SFC leaf of the subtree
    ref = brute_first_leaf_owner(f, own)
    for lc in cells:
        for g, o in zip(lc.gc, lc.owner):
            assert ref[(lc.level, tuple(int(v) for v in g))] == o
    assert all(m.Nlp[l].sum() == m.N[l] for l in range(L + 1))


def test_W0_override():
    f = fig2_forest(2)
    cells = Pt.level_cells(f, Pt.leaf_owners(f, 3))
    m = Pt.model(cells, 3, W0_override=5)
    assert m.W == 5 + 3 + 2 and m.W_sync == 5 + 2 + 2
    assert m.W_opt == Fraction(5 + 8, 3)
