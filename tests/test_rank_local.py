"""Rank-local topology (GMG_RANK_LOCAL, csrc/local_direct.cpp): each rank builds
only its families, the families of the parents of its next-finer families and
their vertex neighbours (only the mesh parts relevant to a processor
are stored; ownership is available without global communication).  It must
produce exactly the rank-local layout the global numbering yields (make_local):
owned/ghost keys and order, ghost owners, exchange plans, cell and transfer
tables in local indices, classes, lambda slots, the key-based eigen start vector
(R10b) and the leaf DoFs -- for every rank, both partition rules, 2D and 3D,
Q1 and Q2.  CPU only (GMG_HOST_ONLY)."""
import numpy as np
import pytest

import paper_1904_03317_b200 as G
from gmg_inputs import config

CASES = [("c1", 1, "first_child", (1, 2, 5)), ("c1", 2, "first_child", (3, 8)),
         ("c3p2", 2, "first_child", (1, 2, 3, 8)), ("c3p2", 1, "first_child", (4, 7)),
         ("c3p2", 2, "per_level", (3, 6)), ("c4s", 2, "first_child", (2, 5)), ("c4s", 2, "per_level", (4,)),
         ("brick8", 2, "first_child", (3, 5)), ("brick8", 1, "per_level", (5,)), ("c2p", 2, "first_child", (3,))]


def _cfg(name):
    if name == "c4s":
        cfg = config("c4")
        cfg.update(s=2, lmax=7)
        return cfg, -1
    if name == "c3p2":
        return config("c3"), 2
    if name == "c2p":                          # the L-shape config at a small depth
        cfg = config("c2")
        cfg.update(lmax=7)
        return cfg, -1
    return config(name), -1


@pytest.mark.parametrize("name,k,mode,ps,coarse", [c + (0,) for c in CASES] +
                         [("c3p2", 2, "first_child", (3, 8), 600), ("c4s", 2, "per_level", (4,), 100)])
def test_rank_local_equals_global_layout(name, k, mode, ps, coarse):
    cfg, passes = _cfg(name)
    f = G.gmg_forest_generate(G.recipe_from_config(cfg, passes))
    for p in ps:
        part = G.gmg_partition(f, p, mode=mode, coarse_cells=coarse)
        for r in range(p):
            hg = G.gmg_setup(f, part, k=k, rank=r, host_only=True, eig_key=True)
            hl = G.gmg_setup(f, part, k=k, rank=r, host_only=True, rank_local=True)
            n_levels = hg.info()["n_levels"]
            for l in range(n_levels):
                a, b = hg.local_level(l), hl.local_level(l)
                for key in a:
                    assert np.array_equal(a[key], b[key]), (p, r, l, key)
                ta, tb = hg.local_tables(l), hl.local_tables(l)
                for key in ta:
                    assert np.array_equal(ta[key], tb[key]), (p, r, l, key)
            ka, kb = hg.owned_leaf_keys(), hl.owned_leaf_keys()
            assert np.array_equal(ka[0], kb[0]) and np.array_equal(ka[1], kb[1]), (p, r)


def test_rank_local_single_rank_sizes():
    """With one rank the summed counts are the global sizes of the global build."""
    cfg = config("c3")
    f = G.gmg_forest_generate(G.recipe_from_config(cfg, 2))
    part = G.gmg_partition(f, 1)
    ig = G.gmg_setup(f, part, k=2, host_only=True).info()
    il = G.gmg_setup(f, part, k=2, host_only=True, rank_local=True).info()
    for key in ("n_leaf_nodes", "n_leaf_free", "n_leaf_hanging", "n_leaf_dirichlet", "n_owned", "first_owned",
                "level_dofs", "level_cells", "level_families", "level_S", "level_E", "level_B", "level_leaf_cells"):
        assert ig[key] == il[key], key


def test_rank_local_global_exports_refused():
    cfg = config("c1")
    f = G.gmg_forest_generate(G.recipe_from_config(cfg))
    part = G.gmg_partition(f, 2)
    h = G.gmg_setup(f, part, k=1, rank=1, host_only=True, rank_local=True)
    with pytest.raises(G.GmgError):
        h.level_dofs(1)
    with pytest.raises(G.GmgError):
        h.leaf_dofs()
