"""Bit-exact integer parity of libgmg's host layer (forest, closure, partition,
model, level numbering, classes, cell tables, lambda map, leaf numbering)
against the oracle, for simulated rank counts, plus the C-ABI symbol check.
CPU only (GMG_HOST_ONLY): no compute call needs a GPU here."""
import ctypes
import os
import re
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_1904_03317_b200 as G
from oracle import forest as F, partition as Pt, mg
from gmg_inputs import config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ ABI
def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "gmg.h")).read()
    decl = set(re.findall(r"\b(gmg_[a-z0-9_]+)\s*\(", hdr))
    lib = ctypes.CDLL(G.LIB_PATH)
    missing = [s for s in sorted(decl) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(G.EXPORTED) <= decl
    assert lib.gmg_abi_version() == 2


# ------------------------------------------------------------------ helpers
def oracle_leaves_as_abi(f):
    """(tree index, level, morton within tree) of oracle leaves."""
    tree = f.tree_index()
    tpos = f.gc >> f.level[:, None]
    loc = f.gc - (tpos << f.level[:, None])
    mor = F.morton(loc, 32).astype(np.uint64)
    return tree.astype(np.int32), f.level.astype(np.int8), mor


def compare_forest(lib_forest, f):
    lt, ll, lm = lib_forest.leaves()
    ot, ol, om = oracle_leaves_as_abi(f)
    assert np.array_equal(lt, ot) and np.array_equal(ll, ol) and np.array_equal(lm, om)


def compare_partition(part, f, p):
    own = Pt.leaf_owners(f, p)
    cells = Pt.level_cells(f, own)
    for lc in cells:
        key, o, leaf = part.level_cells(lc.level)
        assert np.array_equal(key.astype(np.int64), F.morton(lc.gc, 32))
        assert np.array_equal(o, lc.owner) and np.array_equal(leaf.astype(bool), lc.is_leaf)
    m = Pt.model(cells, p)
    lm = part.model()
    assert Fraction(*lm["W_opt"]) == m.W_opt and lm["W_sync"] == m.W_sync and lm["W"] == m.W
    assert Fraction(*lm["eta"]) == m.eta
    assert lm["N"] == list(m.N) and lm["W_l"] == list(m.W_l)
    assert np.array_equal(part.tallies(), m.Nlp)
    g, t = Pt.ghost_children(cells)
    assert lm["ghost_children"] == list(g) and lm["children"] == list(t)
    return cells


def compare_topology(h, f, k, p):
    T = mg.topology(f, k, p)
    info = h.info()
    for l, s in enumerate(T.spaces):
        key, cls, own, can = h.level_dofs(l)
        go = s.global_order()
        assert np.array_equal(key.astype(np.int64), s.key[go])
        assert np.array_equal(cls, s.cls[go])
        assert np.array_equal(own, s.owner[go])
        assert np.array_equal(can, go)
        # cell -> DoF table (global indices), Dirichlet = -1
        inv = np.empty(max(s.n, 1), dtype=np.int64)
        inv[go] = np.arange(s.n)
        ocd = np.where(s.cell_dofs >= 0, inv[np.maximum(s.cell_dofs, 0)], -1)
        assert np.array_equal(h.cell_dofs(l), ocd)
        assert info["level_B"][l] == s.n_boundary
    key, lam, own, can = h.leaf_dofs()
    lf = T.leaf
    fkey = lf.key[lf.free_index >= 0]
    assert np.array_equal(key.astype(np.int64), fkey[T.leaf_global])
    assert np.array_equal(lam, lf.lam[T.leaf_global])
    assert np.array_equal(own, T.leaf_owner[T.leaf_global])
    assert np.array_equal(can, T.leaf_global)
    assert info["n_leaf_nodes"] == lf.X.shape[0]
    assert info["n_leaf_hanging"] == int(lf.hanging.sum())
    assert info["n_leaf_dirichlet"] == int(lf.dirichlet.sum())


# ------------------------------------------------------------------ tests
def test_config1_all_ranks():
    cfg = config("c1")
    f = F.generate(cfg)
    lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
    compare_forest(lf, f)
    for p in (1, 2, 3, 5, 8):
        part = G.gmg_partition(lf, p)
        compare_partition(part, f, p)
        h = G.gmg_setup(lf, part, k=1, host_only=True)
        compare_topology(h, f, 1, p)


@pytest.mark.parametrize("name,k", [("c1", 2), ("c3p2", 2), ("c3p2", 1)])
def test_small_configs_topology(name, k):
    cfg = config(name)
    f = F.generate(cfg)
    lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
    compare_forest(lf, f)
    for p in (1, 4, 7):
        part = G.gmg_partition(lf, p)
        compare_partition(part, f, p)
        h = G.gmg_setup(lf, part, k=k, host_only=True)
        compare_topology(h, f, k, p)


def test_lshape_multitree_topology():
    cfg = dict(config("c2"))
    cfg["lmax"] = 7
    cfg["s"] = 2
    f = F.generate(cfg)
    lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
    compare_forest(lf, f)
    for p in (1, 3):
        part = G.gmg_partition(lf, p)
        compare_partition(part, f, p)
        h = G.gmg_setup(lf, part, k=2, host_only=True)
        compare_topology(h, f, 2, p)


@pytest.mark.slow
def test_config2_topology_full():
    cfg = config("c2")
    f = F.generate(cfg)
    lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
    compare_forest(lf, f)
    part = G.gmg_partition(lf, 2)
    compare_partition(part, f, 2)
    h = G.gmg_setup(lf, part, k=2, host_only=True)
    compare_topology(h, f, 2, 2)


@settings(max_examples=15, deadline=None)
@given(st.integers(2, 3), st.integers(1, 2), st.lists(st.integers(0, 10 ** 6), min_size=1, max_size=5),
       st.integers(1, 6))
def test_random_forests_create_and_topology(d, k, picks, p):
    f = F.coarse_forest(d, [(0,) * d])
    f = F.refine(f, np.ones(1, dtype=bool))
    for q in picks:
        m = np.zeros(f.n_leaves, dtype=bool)
        m[q % f.n_leaves] = True
        f = F.close(F.refine(f, m))
        if f.n_leaves > 250:
            break
    t, l, mo = oracle_leaves_as_abi(f)
    lf = G.gmg_forest_create(d, [(0,) * d], t, l, mo)
    compare_forest(lf, f)
    part = G.gmg_partition(lf, p)
    compare_partition(part, f, p)
    h = G.gmg_setup(lf, part, k=k, host_only=True)
    compare_topology(h, f, k, p)


def test_forest_create_validation_and_closure():
    # unbalanced forest: rejected, or closed equal to the oracle closure
    f = F.coarse_forest(2, [(0, 0)])
    f = F.refine(F.refine(f, [True]), np.ones(4, dtype=bool))
    m = np.zeros(f.n_leaves, dtype=bool)
    m[0] = True
    f = F.refine(f, m)
    m = (f.level == 3) & np.all(f.gc == 1, axis=1)
    f = F.refine(f, m)
    t, l, mo = oracle_leaves_as_abi(f)
    with pytest.raises(G.GmgError) as e:
        G.gmg_forest_create(2, [(0, 0)], t, l, mo)
    assert e.value.code == 4                                  # GMG_E_UNBALANCED
    lf = G.gmg_forest_create(2, [(0, 0)], t, l, mo, flags=G.GMG_CLOSE_BALANCE)
    compare_forest(lf, F.close(f))
    # unsorted
    with pytest.raises(G.GmgError) as e:
        G.gmg_forest_create(2, [(0, 0)], t[::-1].copy(), l[::-1].copy(), mo[::-1].copy())
    assert e.value.code == 2
    # hole
    with pytest.raises(G.GmgError) as e:
        G.gmg_forest_create(2, [(0, 0)], t[1:], l[1:], mo[1:])
    assert e.value.code == 3
    # bad args
    with pytest.raises(G.GmgError) as e:
        G.gmg_forest_create(4, [(0, 0, 0, 0)], t, l, mo)
    assert e.value.code == 1
    lf = G.gmg_forest_create(2, [(0, 0)], np.zeros(1), np.zeros(1), np.zeros(1))
    with pytest.raises(G.GmgError) as e:
        G.gmg_partition(lf, 0)
    assert e.value.code == 1


def test_fig2_through_abi():
    """The paper's worked example through the C ABI: W_opt=3, W_sync=5, W=6,
    eta=1/2."""
    f = F.coarse_forest(2, [(0, 0)])
    f = F.refine(f, [True])
    m = np.zeros(4, dtype=bool)
    m[2] = True
    f = F.refine(f, m)
    t, l, mo = oracle_leaves_as_abi(f)
    lf = G.gmg_forest_create(2, [(0, 0)], t, l, mo)
    mod = G.gmg_partition(lf, 3).model()
    assert Fraction(*mod["W_opt"]) == 3 and mod["W_sync"] == 5 and mod["W"] == 6
    assert Fraction(*mod["eta"]) == Fraction(1, 2)
    assert G.gmg_partition(lf, 3).model(W0_override=5)["W"] == 10
